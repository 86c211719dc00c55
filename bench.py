#!/usr/bin/env python3
"""Benchmark: 16x16 S-box full fused nonlinearity on B200 (BASELINE.json metric).

One step = one pass of the hot path over one S-box: for all 65535 output
masks, generate the +/-1 component from the table, run the length-2^16
integer FWHT, fold max|W| (sbw_nl, one fused kernel) and convert to
per-component NL (sbw_maxabs_to_nl).  Inputs are resident in HBM when the
timed region starts; L2 is flushed (256 MiB write) between timed steps and
every step is timed with its own CUDA events on the launching stream.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config 16x16|12x12|20x20|24x16]

Multi-GPU (torchrun): weak scaling -- every rank evaluates its own full
16x16 box (seed = rank); no collective on the data path; time = max over
ranks.  --shard (the north_star's mode for 20x20 / 24x16): strong scaling --
one box (seed 0), rank r evaluates the masks partition_columns(2^m-1, N)[r]
(parallel.py:38-57) and each step ends with the path's one exchange, an
all_reduce(MAX) of the 8-byte (max|W|, smallest v) key.  --impl reference times the reference's CPU algorithm (the oracle
port of its per-mask stream loop, walsh.py:230-244) on all host cores over a
bounded sample of masks and prints the same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {  # name -> (n, m, bijective)   BASELINE.json configs
    "8x8": (8, 8, True),
    "12x12": (12, 12, True),
    "16x16": (16, 16, True),
    "20x20": (20, 20, False),
    "24x16": (24, 16, False),
}
# PAPER.md:421 (via BASELINE.md): best published 16x16 full NL = 83,015 ms (fused, CPU)
PAPER_16x16_NL_MS = 83015.0


def coeffs(n, m, masks=None):
    return (masks if masks is not None else (1 << m) - 1) * (1 << n)


# ----------------------------------------------------------------- clocks ---
class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region.

    NVML (pynvml) polls every ~2 ms, so even a ~20 ms timed region gets many
    samples; nvidia-smi is the fallback.
    """

    REASONS = {  # NVML clocks-event-reason bits (nvmlClocksEventReason*)
        "sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, reason bitmask)
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self, nv):
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            try:
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            except AttributeError:
                rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            self.samples.append((float(sm), float(mx), int(rs)))
            self._stop.wait(0.002)

    def _run_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        bits = [0x8, 0x40, 0x20, 0x4]
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5)
                f = [x.strip() for x in out.stdout.strip().split(",")]
                mask = sum(b for b, v in zip(bits, f[2:6]) if v.lower() == "active")
                self.samples.append((float(f[0]), float(f[1]), mask))
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.05)

    def _run(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            try:
                self._run_nvml(nv)
            finally:
                nv.nvmlShutdown()
        except Exception:  # noqa: BLE001
            self._run_smi()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.01)  # first sample before the timed work starts
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [s[0] for s in self.samples]
        mask = 0
        for s in self.samples:
            mask |= s[2]
        reasons = sorted(k for k, b in self.REASONS.items() if mask & b)
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------ CPU baseline --
def _cpu_worker(args):
    n, m, bij, lo, hi = args
    from oracle import sbw_oracle as orc

    t = orc.gen_table(n, m, 0, bij)
    t0 = time.perf_counter()
    orc.stream_loop(t, n, lo, hi)
    return time.perf_counter() - t0


def cpu_baseline(name, target_s=12.0, procs=None):
    """Reference CPU algorithm (oracle port of walsh.py:230-244) on all host
    cores over a bounded mask sample; returns coeff/s and a description."""
    import multiprocessing as mp

    from oracle import sbw_oracle as orc

    n, m, bij = CONFIGS[name]
    procs = procs or os.cpu_count() or 1
    t = orc.gen_table(n, m, 0, bij)
    # calibrate one core on a few masks
    k0 = 4 if n >= 20 else 16
    t0 = time.perf_counter()
    orc.stream_loop(t, n, 1, 1 + k0)
    per_mask = (time.perf_counter() - t0) / k0
    per_proc = max(1, int(target_s / per_mask / 2))
    total = min((1 << m) - 1, per_proc * procs)
    part = orc.partition_columns(total, procs)
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(len(part)) as pool:
        pool.map(_cpu_worker, [(n, m, bij, a, b) for a, b in part])
    wall = time.perf_counter() - t0
    value = coeffs(n, m, total) / wall
    return {"value": value, "unit": "coeff/s", "cores": len(part), "kind": "port",
            "sample": f"{name} seed 0, masks 1..{total} of {(1 << m) - 1}, reference per-mask "
                      f"stream loop (oracle port of walsh.py:230-244) in {len(part)} processes, "
                      f"{wall:.1f} s wall"}


def cpu_engine(name, target_s=4.0):
    """The reference's SHIPPED engine shape: fwht_parallel
    (parallel.py:64-133) = a ThreadPoolExecutor over partition_columns ranges,
    each worker running the per-mask stream body (walsh.py:237-240), here the
    oracle port of that body.  Timed with workers = os.cpu_count() and 1 over
    a bounded mask sample; the GIL lets ~1 core run numpy's small per-stage
    ufunc calls at a time, which is why the process harness above is faster."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import sbw_oracle as orc

    n, m, bij = CONFIGS[name]
    t = orc.gen_table(n, m, 0, bij)
    k0 = 2 if n >= 20 else 8
    t0 = time.perf_counter()
    orc.stream_loop(t, n, 1, 1 + k0)
    per_mask = (time.perf_counter() - t0) / k0
    total = max(1, min((1 << m) - 1, int(target_s / per_mask / 2)))
    out = {"sample": f"{name} seed 0, masks 1..{total}", "unit": "coeff/s",
           "note": "reference engine shape: ThreadPoolExecutor(workers) over partition_columns "
                   "ranges running the per-mask stream body (oracle port); GIL-bound"}
    for workers in (os.cpu_count() or 1, 1):
        part = orc.partition_columns(total, workers)
        t0 = time.perf_counter()
        with ThreadPoolExecutor(max_workers=len(part)) as pool:
            list(pool.map(lambda r: orc.stream_loop(t, n, r[0], r[1]), part))
        out[f"workers_{workers}"] = coeffs(n, m, total) / (time.perf_counter() - t0)
    out["cores"] = os.cpu_count() or 1
    return out


# ------------------------------------------------------------------- GPU ----
def measured_hbm_peak():
    """HBM copy bandwidth in GB/s from the driver-written MEASURED_PEAKS.json,
    else the fallback B200_PROFILING.md states."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (driver-measured copy)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback 6.65 TB/s of B200_PROFILING.md (MEASURED_PEAKS.json absent)"


def live_peak(lib, d, fn):
    """Best of 2 runs of a libsbw peak microbenchmark (sbw_int32_peak / sbw_int8_mma_peak)."""
    import ctypes

    best = 0.0
    for _ in range(2):
        ops, ms = ctypes.c_double(0), ctypes.c_double(0)
        d.check(getattr(lib, fn)(ctypes.byref(ops), ctypes.byref(ms), None))
        best = max(best, ops.value)
    return best


def run_ours(args, rank, world, local_rank):
    import torch

    import paper_1912_03732_b200 as sw
    from paper_1912_03732_b200 import device as d

    # SBW_BENCH_BACKEND=gloo (plumbing check only): several ranks may share a
    # GPU, which NCCL refuses; the timing of such a run means nothing.
    backend = os.environ.get("SBW_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local_rank = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    lib = d.load_library()
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def barrier():
        if dist is not None:
            dist.barrier()

    n, m, bij = CONFIGS[args.config]
    s = sw.generate_sbox(n, m, seed=0 if args.shard else rank, bijective=bij)
    v_lo, v_hi = 1, 1 << m
    if args.masks:
        v_hi = min(v_hi, 1 + args.masks)
    total_masks = v_hi - v_lo
    if args.shard:  # this rank's contiguous balanced mask range
        v_lo, v_hi = sw.partition_columns(total_masks, world).ranges[rank]
    nmask = v_hi - v_lo
    tab = d.device_table(s, dev, cache=False)
    mx = torch.empty(nmask, dtype=torch.int32, device=dev)
    key = torch.zeros(1, dtype=torch.int64, device=dev)
    nl = torch.empty(nmask, dtype=torch.int64, device=dev)
    bad = torch.empty(1, dtype=torch.int64, device=dev)
    sbytes = lib.sbw_nl_scratch_bytes(n, m, v_lo, v_hi)
    scratch = torch.empty(max(1, sbytes), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream
    tb = d.table_bytes(m)

    def step():
        key.zero_()
        d.check(lib.sbw_nl(tab.data_ptr(), tb, n, m, v_lo, v_hi, mx.data_ptr(), key.data_ptr(),
                           scratch.data_ptr(), sbytes, sh))
        d.check(lib.sbw_maxabs_to_nl(mx.data_ptr(), nmask, n, nl.data_ptr(), bad.data_ptr(), sh))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    # ---- timed region: K steps, per-step events, L2 flushed in between ----
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    launches0 = d.launch_count()
    barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            evs[i][0].record(stream)
            key.zero_()
            kev[i][0].record(stream)
            d.check(lib.sbw_nl(tab.data_ptr(), tb, n, m, v_lo, v_hi, mx.data_ptr(),
                               key.data_ptr(), scratch.data_ptr(), sbytes, sh))
            kev[i][1].record(stream)
            d.check(lib.sbw_maxabs_to_nl(mx.data_ptr(), nmask, n, nl.data_ptr(), bad.data_ptr(),
                                         sh))
            if args.shard and dist is not None:  # the path's exchange: global (max|W|, v) key
                dist.all_reduce(key, op=dist.ReduceOp.MAX)
            evs[i][1].record(stream)
        torch.cuda.synchronize(dev)
    barrier()
    launches = d.launch_count() - launches0
    step_ms = sum(a.elapsed_time(b) for a, b in evs)
    kern_ms = sum(a.elapsed_time(b) for a, b in kev) / args.steps
    if dist is not None:
        t = torch.tensor([step_ms, kern_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms, kern_ms = float(t[0]), float(t[1])

    # ---- correctness of what was timed (against the committed goldens) ----
    if int(bad.item()) != (1 << 63) - 1:
        raise AssertionError("odd spectrum gap in the benchmark run")
    res = sw.walsh.decode_key(key, n)
    check = {"nl": res[0], "argmin_v": res[1], "max_abs": res[2]}
    if args.config == "16x16" and rank == 0 and not args.masks and (args.shard or world == 1):
        assert (res[0], res[1]) == (31942, 44828), res

    # ---- e2e through the C ABI with host buffers (sbw_nl_host) ------------
    # The caller's table and result buffers are page-locked once
    # (cudaHostRegister), as a repeated caller would: sbw_nl_host then DMAs
    # them directly, every step, inside the timed region.
    h_nl = np.empty(nmask, dtype=np.int64)
    out3 = np.empty(3, dtype=np.int64)
    table_host = np.ascontiguousarray(s.table)
    cudart = torch.cuda.cudart()
    registered = []
    for arr in (table_host, h_nl):
        if int(cudart.cudaHostRegister(arr.ctypes.data, arr.nbytes, 0)) == 0:
            registered.append(arr)
    for _ in range(2):
        d.check(lib.sbw_nl_host(table_host.ctypes.data, n, m, v_lo, v_hi, h_nl.ctypes.data,
                                out3.ctypes.data, local_rank))
    barrier()
    t0 = time.perf_counter()
    gkey = torch.zeros(1, dtype=torch.int64, device=dev)
    for _ in range(args.steps):
        d.check(lib.sbw_nl_host(table_host.ctypes.data, n, m, v_lo, v_hi, h_nl.ctypes.data,
                                out3.ctypes.data, local_rank))
        if args.shard and dist is not None:  # combine the shards' (max|W|, argmin v)
            gkey.fill_((int(out3[2]) << 32) | (0xFFFFFFFF - int(out3[1])))
            dist.all_reduce(gkey, op=dist.ReduceOp.MAX)
            int(gkey.item())
    e2e_s = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t[0])
    assert np.array_equal(h_nl, nl.cpu().numpy())
    for arr in registered:
        cudart.cudaHostUnregister(arr.ctypes.data)

    # ---- roofline of the dominant kernel (fused NL) ----------------------
    peak = live_peak(lib, d, "sbw_int32_peak")
    clk_summary = clk.summary()
    dual_issue = (2 * 4 * 32 * d.device_info(local_rank)["sm_count"]
                  * (clk_summary["sm_max_mhz"] or 1965) * 1e6)  # packed-16x2 lane-ops/s, both int pipes
    # sbw_nl takes the tensor-core kernel for n = 12..16 (n < 16: 2^(16-n)
    # components per 2^16 tile; needs m >= 16 - n), unless SBW_TC=0
    tc_path = 12 <= n <= 16 and m >= 16 - n and os.environ.get("SBW_TC", "1") != "0"
    prof = os.path.join(ROOT, "profiles", f"ncu_{args.config}_traffic.json")
    traffic = None
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    if tc_path:
        # k_tc_hybrid<NL>: the r stages (x bits 0..7) run as an int8 GEMM on
        # the tensor cores; the c stages (x bits 8..15) run on the integer
        # ALUs -- 4 of them as byte-lane butterflies on the bit rows of the
        # GEMM's B operand (c bits 0..3, inside the generation), 4 as packed
        # 16-bit stages after the GEMM (c bits 4..7, incl. the max fold).  The
        # integer half is the limiter (ALU pipe ~80 %), so it is the primary
        # roofline: 8 stages x 2^16 butterfly element-ops per component
        # against the packed-16x2 rate (2 x the live int32 lane-op peak; the
        # byte-lane stages would allow 4x, so this is conservative).  The GEMM
        # half is reported beside it: 2 * 256 (M) * 256 (N) * 288 (K incl. the
        # bias block) int8 ops executed per component against the live
        # kind::i8 peak.
        peak_i8 = live_peak(lib, d, "sbw_int8_mma_peak")
        lc = 16 - n
        items = ((v_hi - 1) >> lc) + 1 - (v_lo >> lc)  # 2^16 tiles
        alu_ops = (n - 8) * (1 << n) * nmask
        mma_ops = 2 * 256 * 256 * 288 * items
        achieved = alu_ops / (kern_ms * 1e-3)
        # n = 16 (unless SBW_TC_LUT=0): k_tc_lut16, the GEMM contracts x bits
        # 8..15 and the other 8 stages are 3 by table lookup (byte -> 8-point
        # WHT, LDS.64), 4 as byte-lane butterflies and the top one on packed
        # int16 lanes with the max fold.  The GEMM half is the primary
        # roofline there (18 MMAs per component against the live kind::i8
        # rate; ncu: issue slots 92 %, ALU pipe 70 %, tensor pipe active 66 %)
        # and the integer half sits beside it under "integer".
        lut = n == 16 and os.environ.get("SBW_TC_LUT", "1") != "0"
        kernel_name = (
            "k_tc_lut16 (tcgen05 int8 GEMM over x bits 8..15; x bits 0..7: 3 stages by shared-memory "
            "table lookup, 4 byte-lane stages on the GEMM operand, the top stage + max fold on packed "
            "int16 lanes)" if lut else
            f"k_tc_hybrid<NL, {n}> (tcgen05 int8 GEMM over x bits 0..7; x bits 8..{n - 1} on "
            "the integer ALUs: 4 byte-lane stages on the GEMM operand + packed int16 stages)")
        roofline = {
            "bound": "int32_alu",
            "kernel": kernel_name,
            "achieved": achieved / 1e12, "peak": 2 * peak / 1e12, "unit": "Tops/s",
            "frac": achieved / (2 * peak), "traffic": traffic,
            "ops_per_launch": alu_ops,
            "ops_definition": "integer half: (n-8) stages x 2^n butterfly element-ops per component "
                              "(x bits 8..n-1: 4 byte-lane + n-12 int16-lane stages incl. the "
                              "max fold); the r stages run as the int8 GEMM below",
            "kernel_ms": kern_ms,
            "peak_source": "measured live by sbw_int32_peak (best of IADD3/LOP3, IMAD and mixed "
                           "chains, int32 lane-ops/s) x 2 lanes for packed 16-bit; not in "
                           "MEASURED_PEAKS.json",
            "peak_dual_issue": dual_issue / 1e12,
            "frac_dual_issue": achieved / dual_issue,
            "peak_dual_issue_source": "theoretical: 4 warp-instr/clk/SM (ALU + FMA pipes dual-issued) "
                                      "x 32 lanes x SMs x max SM clock x 2 packed 16-bit lanes",
            "tensor": {"achieved": mma_ops / (kern_ms * 1e-3) / 1e15, "peak": peak_i8 / 1e15,
                       "unit": "POP/s int8", "frac": mma_ops / (kern_ms * 1e-3) / peak_i8,
                       "ops_per_launch": mma_ops,
                       "peak_source": "measured live by sbw_int8_mma_peak (tcgen05.mma.kind::i8 "
                                      "128x256x32 chains, one CTA per SM)"},
            "whole_fwht_equiv": {"ops_per_launch": n * (1 << n) * nmask,
                                 "achieved": n * (1 << n) * nmask / (kern_ms * 1e-3) / 1e12,
                                 "unit": "T butterfly element-ops/s",
                                 "vs_int32_alu_peak": n * (1 << n) * nmask / (kern_ms * 1e-3) / peak,
                                 "vs_packed16_alu_peak": n * (1 << n) * nmask / (kern_ms * 1e-3)
                                 / (2 * peak)},
        }
        if lut:
            # primary: the tensor pipe; "integer" keeps the previous primary numbers
            integer = {k: roofline[k] for k in ("achieved", "peak", "unit", "frac", "ops_per_launch",
                                                "ops_definition", "peak_source", "peak_dual_issue",
                                                "frac_dual_issue", "peak_dual_issue_source")}
            integer["ops_definition"] = (
                "integer half: 8 stages x 2^16 butterfly element-ops per component (x bits 0..7: "
                "3 by table lookup, 4 byte-lane, 1 int16-lane stage incl. the max fold) against the "
                "packed-16x2 ALU rate")
            t = roofline["tensor"]
            roofline = {
                "bound": "tensor", "kernel": kernel_name,
                "achieved": t["achieved"], "peak": t["peak"], "unit": t["unit"], "frac": t["frac"],
                "traffic": traffic, "ops_per_launch": t["ops_per_launch"],
                "ops_definition": "GEMM half: 2 * 256 (M) * 256 (N) * 288 (K: x bits 8..15 + the bias "
                                  "block) int8 ops per component, 8 of the 16 stages",
                "kernel_ms": kern_ms, "peak_source": t["peak_source"],
                "integer": integer, "whole_fwht_equiv": roofline["whole_fwht_equiv"],
                # what actually binds the kernel (K2L): one 128-byte
                # shared-memory wavefront per clock per SM, shared by the tensor
                # core's operand fetch (18 MMAs x (4 + 8) KiB) and the generation
                # (64 KiB of table lookups + 64 KiB of B-operand stores)
                "shared_memory": {
                    "bytes_per_component": (18 * 12 + 64 + 64) * 1024,
                    "achieved": (18 * 12 + 64 + 64) * 1024 * items / (kern_ms * 1e-3) / 1e12,
                    "peak": 128 * d.device_info(local_rank)["sm_count"]
                    * (clk_summary["sm_max_mhz"] or 1965) * 1e6 / 1e12,
                    "unit": "TB/s",
                    "frac": (18 * 12 + 64 + 64) * 1024 * items / (kern_ms * 1e-3)
                    / (128 * d.device_info(local_rank)["sm_count"] * (clk_summary["sm_max_mhz"] or 1965) * 1e6),
                    "peak_source": "128 B/clk/SM x SMs x max SM clock (ncu: tc + lsu shared wavefronts "
                                   "per component = cycles per component, profiles/r2_ncu_16x16_k_tc_lut16.md)",
                },
            }
    elif n >= 17:
        # Multi-pass K3: pass A (k_tc_hybrid<emit>) writes every component's
        # stage-15 partial transform as u16 and pass B reads it back -- 4 B of
        # HBM traffic per element, the bound once pass A runs on the tensor
        # cores.  Peak: the driver-measured HBM copy bandwidth.
        hbm_peak, hbm_src = measured_hbm_peak()
        alg_bytes = 4 * (1 << n) * nmask
        alg_ops = n * (1 << n) * nmask
        roofline = {"bound": "hbm", "kernel": "k3: k_tc_hybrid<emit> (pass A) + k_passb (pass B)",
                    "achieved": alg_bytes / (kern_ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                    "frac": alg_bytes / (kern_ms * 1e-3) / 1e9 / hbm_peak, "traffic": traffic,
                    "bytes_per_launch": alg_bytes,
                    "bytes_definition": "u16 scratch written by pass A and read by pass B: 2 + 2 B per "
                                        "element per component",
                    "kernel_ms": kern_ms, "peak_source": hbm_src,
                    "int32_alu": {"achieved": alg_ops / (kern_ms * 1e-3) / 1e12, "peak": peak / 1e12,
                                  "unit": "Tops/s", "frac": alg_ops / (kern_ms * 1e-3) / peak,
                                  "ops_definition": "n * 2^n butterfly element-ops per component"}}
    else:
        alg_ops = n * (1 << n) * nmask  # butterfly element-ops
        achieved = alg_ops / (kern_ms * 1e-3)
        # The kernel's butterflies run on packed 16-bit (and 8-bit) integer
        # lanes, two or four per 32-bit instruction, so the denominator is the
        # packed-16x2 rate: 2 x the measured int32 lane-op peak (same
        # instruction issue rate, two lanes each).  frac_int32 is the same
        # number against the plain int32 peak (can exceed 1 because of packing).
        roofline = {"bound": "int32_alu",
                    "kernel": "k_tile_simd",
                    "achieved": achieved / 1e12, "peak": 2 * peak / 1e12, "unit": "Tops/s",
                    "frac": achieved / (2 * peak), "traffic": traffic,
                    "peak_int32": peak / 1e12, "frac_int32": achieved / peak,
                    "ops_per_launch": alg_ops, "ops_definition": "n * 2^n butterfly element-ops "
                    "per component (SURVEY.md 8d)", "kernel_ms": kern_ms,
                    "peak_source": "measured live by sbw_int32_peak (IADD3/LOP3 + IMAD chains, "
                                   "int32 lane-ops/s) x 2 lanes for packed 16-bit; "
                                   "not in MEASURED_PEAKS.json"}

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    total_coeff = coeffs(n, m, total_masks if args.shard else nmask * world) * args.steps
    value = total_coeff / (step_ms * 1e-3)
    line = {
        "metric": f"Walsh coefficients/s, {args.config} S-box full fused nonlinearity "
                  "(all 2^m-1 components, max|W| and per-component NL)",
        "value": value,
        "unit": "coeff/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": step_ms / args.steps,
        "full_nl_ms": step_ms / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if args.shard else "weak",
        "vs_baseline": (value / (1 if args.shard else world)) / (coeffs(16, 16) / (PAPER_16x16_NL_MS * 1e-3))
        if args.config == "16x16" and not args.masks else None,
        "vs_baseline_ref": "PAPER.md:421 fused NL 16x16 = 83,015 ms on i7-8700K-class CPU (BASELINE.md)",
        "dtype": ("int8 MMA (s32 acc) + packed int16" if tc_path else
                  ("u16 scratch: int8 MMA pass A (s32 acc), pass B "
                   + ("int8 MMA (s32 acc)" if n >= 21 else "fp32 (exact integers < 2^24)"))
                  if n >= 17 else "packed int8/int16 lanes (int32 ALU)"),
        "data": "synthetic: generate_sbox(n, m, seed=rank) -- numpy PCG64 like the reference",
        "config": {"workload": f"{args.config} S-box (n={n}, m={m}, bijective={bij}), "
                               f"masks [{v_lo},{v_hi}), full NL per step",
                   "parallelism": (f"strong x{world} (masks sharded by partition_columns, "
                                   "all_reduce(MAX) of the key per step)") if args.shard
                                  else f"weak x{world} (one S-box per GPU)",
                   "l2": "flushed between timed steps (256 MiB write), per-step CUDA events"},
        "result": check,
        "roofline": roofline,
        "e2e": {"value": coeffs(n, m, total_masks if args.shard else nmask * world) * args.steps / e2e_s,
                "unit": "coeff/s",
                "h2d_bytes_per_step": int(table_host.nbytes),  # uint32 table
                "d2h_bytes_per_step": int(h_nl.nbytes + 8 * 4),
                "path": "sbw_nl_host C ABI (host table in, host NL out, page-locked caller "
                        "buffers), wall clock"},
        "gpu_launches": int(launches),
        "clocks": clk_summary,
    }
    if not args.no_cpu and world == 1:  # the CPU baseline is reported at N = 1 only
        line["cpu_baseline"] = cpu_baseline(args.config, target_s=args.cpu_seconds)
        line["cpu_baseline"]["engine"] = cpu_engine(args.config, target_s=args.cpu_seconds / 3)
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def run_reference(args, rank, world):
    if rank != 0:
        return
    n, m, bij = CONFIGS[args.config]
    vals = []
    base = None
    for _ in range(args.warmup):
        cpu_baseline(args.config, target_s=args.cpu_seconds / 4)
    for _ in range(args.steps):
        base = cpu_baseline(args.config, target_s=args.cpu_seconds)
        vals.append(base["value"])
    value = statistics.mean(vals)
    full_s = coeffs(n, m) / value
    line = {
        "impl": "reference",
        "metric": f"Walsh coefficients/s, {args.config} S-box full fused nonlinearity "
                  "(all 2^m-1 components, max|W| and per-component NL)",
        "value": value, "unit": "coeff/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": full_s * 1e3, "full_nl_ms": full_s * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int32", "data": "synthetic: generate_sbox(n, m, seed=0)",
        "config": {"workload": f"{args.config} S-box (n={n}, m={m}, bijective={bij})",
                   "note": "each step is a bounded mask sample; full-NL time extrapolated "
                           "linearly in the number of masks"},
        "cpu_baseline": dict({k: base[k] for k in ("value", "unit", "cores", "kind", "sample")},
                             engine=cpu_engine(args.config, target_s=args.cpu_seconds / 3)),
        "e2e": {"value": value, "unit": "coeff/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _free_port():
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(n):
    """`python bench.py --gpus N` without torchrun: start N ranks of this
    script (one per GPU, RANK/LOCAL_RANK/WORLD_SIZE/MASTER_* set as torchrun
    would), stream their output, and exit with the worst exit code.  Rank 0
    alone prints the JSON line.  If any rank fails the others are stopped
    (a rank blocked in a collective would otherwise wait forever)."""
    port = _free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:],
                                      env=env))
    rc = 0
    live = list(procs)
    while live:
        for p in list(live):
            code = p.poll()
            if code is None:
                continue
            live.remove(p)
            if code != 0:
                rc = rc or code
                for q in live:
                    q.terminate()
        time.sleep(0.05)
    return rc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=list(CONFIGS), default="16x16")
    ap.add_argument("--masks", type=int, default=0, help="limit masks (debug)")
    ap.add_argument("--shard", action="store_true",
                    help="strong scaling: shard one box's masks over the ranks (the default for N > 1)")
    ap.add_argument("--weak", action="store_true",
                    help="N > 1: one whole box per rank (seed = rank) instead of sharding one box")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    args = ap.parse_args()
    if args.impl == "ours" and "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", args.gpus if args.impl == "reference" else 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    # N > 1: the north_star's mode -- one box, output masks sharded over the
    # GPUs (partition_columns), one max-all-reduce of the key per step
    args.shard = (args.shard or world > 1) and not args.weak
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
