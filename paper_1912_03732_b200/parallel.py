"""Mask-range sharding: the reference's column-parallel engine, GPU-first.

`partition_columns` keeps the reference's balanced contiguous ranges
(parallel.py:38-57).  `fwht_parallel` (parallel.py:64-133) maps those
ranges -- the reference's thread-pool "workers" -- onto the visible GPUs
round-robin as logical shards: every shard is one libsbw launch over its
mask range, results land in disjoint slots, so output is bit-identical for
any shard count.  `evaluate_distributed` is the multi-process form (one rank
per GPU, torch.distributed): each rank owns one range, the per-component
values are all-gathered and the (max|W|, smallest v) key is max-reduced --
the only exchange on the path.  `spectrum_distributed` is the materialised
form: every rank keeps its own range of the Walsh matrix (either layout) on
its GPU and only the key is max-reduced.
"""
from __future__ import annotations

import time

import numpy as np

from . import device as _dev
from .memory import charged, check_budget, memory_estimate
from .records import ColumnMaxima, ColumnPartition, NonlinearityResult, SBox, WalshSpectrum  # noqa: F401
from .walsh import (check_nl_flag, component_max_abs_device, decode_key,  # noqa: F401
                    device_to_host_chunked, maxabs_to_nl, maxabs_to_nl_device, spectrum_device)


def partition_columns(total_columns: int, workers: int) -> ColumnPartition:
    """Split masks 1..total_columns into <= workers balanced contiguous ranges.

    Sizes differ by at most one, the leading ranges take the remainder, and
    more workers than columns degrade to singleton ranges.
    """
    if total_columns < 1:
        raise ValueError(f"total_columns must be >= 1, got {total_columns}")
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    k = min(workers, total_columns)
    q, r = divmod(total_columns, k)
    bounds = [1]
    for i in range(k):
        bounds.append(bounds[-1] + q + (1 if i < r else 0))
    return ColumnPartition(tuple(zip(bounds[:-1], bounds[1:])), workers)


def default_workers() -> int:
    """Default logical shard count: one per visible GPU (at least 1)."""
    try:
        torch = _dev.torch_mod()
        return max(1, torch.cuda.device_count())
    except Exception:  # noqa: BLE001 - no torch/CUDA: still a valid count
        return 1


def _devices():
    torch = _dev.torch_mod()
    _dev.require_device()
    return [torch.device("cuda", i) for i in range(torch.cuda.device_count())]


def fwht_parallel(s: SBox, workers: int | None = None, mode: str = "retain",
                  max_bytes: int | None = None,
                  timings: dict | None = None) -> tuple[WalshSpectrum | None, ColumnMaxima]:
    """Fused transform over `workers` mask-range shards spread across the GPUs.

    Bit-identical to fwht_fused(s, mode) for every shard count.
    """
    if mode not in ("retain", "stream"):
        raise ValueError(f"mode must be 'retain' or 'stream', got {mode!r}")
    if workers is None:
        workers = default_workers()
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    part = partition_columns((1 << s.m) - 1, workers)
    t0 = time.perf_counter()
    if mode == "retain":
        check_budget(((1 << s.m) - 1) * (1 << s.n) * 4, max_bytes)
    else:
        check_budget(memory_estimate(s.n, s.m, mode="stream", workers=len(part.ranges)),
                     max_bytes)
    devs = _devices()
    values = np.empty((1 << s.m) - 1, dtype=np.int64)
    rows = None
    t1 = time.perf_counter()
    pending = []
    nbytes = ((1 << s.m) - 1) * (1 << s.n) * 4 if mode == "retain" else 0
    with charged(nbytes):
        if mode == "retain":
            rows = np.empty(((1 << s.m) - 1, 1 << s.n), dtype=np.int32)
        # every shard is launched (asynchronously, each on its own GPU's
        # current stream) before any result is read back
        for i, (lo, hi) in enumerate(part.ranges):
            dev = devs[i % len(devs)]
            with _dev.on(dev):
                if mode == "retain":
                    spec, mx = spectrum_device(s, lo, hi, layout="mask", device=dev)
                else:
                    spec, (mx, _key) = None, component_max_abs_device(s, lo, hi, device=dev)
            pending.append((lo, hi, spec, mx))
        for lo, hi, spec, mx in pending:  # completion barrier, in range order
            with _dev.on(mx.device):
                values[lo - 1:hi - 1] = maxabs_to_nl(mx, s.n)
                if spec is not None:
                    device_to_host_chunked(spec, rows[lo - 1:hi - 1])
        t2 = time.perf_counter()
    if timings is not None:
        timings["build_s"] = t1 - t0
        timings["transform_s"] = t2 - t1
    spectrum = WalshSpectrum(s.n, s.m, rows) if rows is not None else None
    return spectrum, ColumnMaxima(s.n, s.m, values)


# ---------------------------------------------------------------------------
# multi-process (one rank per GPU) evaluation
# ---------------------------------------------------------------------------
def _gpu_shard(s: SBox, lo: int, hi: int):
    """Default shard compute: fused NL on this rank's GPU, left on the GPU.

    Returns (NL int64 [hi - lo + 1] device tensor whose last entry is the
    odd-gap flag, key int64 [1] device tensor)."""
    mx, key = component_max_abs_device(s, lo, hi)
    return maxabs_to_nl_device(mx, s.n), key


def _evaluate_p2p(s: SBox, group, lo: int, hi: int, total: int,
                  return_values: bool) -> tuple[int, np.ndarray | None]:
    """Peer-memory exchange (sbw_ipc_* / sbw_key_merge, include/sbw.h).

    Rank 0 owns int32 max|W|[2^m - 1] + the uint64 key in IPC-exportable
    device memory; every rank maps them, its sbw_nl stores its component
    maxima straight into rank 0's array (over NVLink when the ranks sit on
    different GPUs) and one system-scope atomicMax folds its key into rank
    0's.  The process group only carries the 64-byte handles and two
    barriers.  Returns (key, per-component NL int64 or None), read back by
    every rank from rank 0's memory.
    """
    import ctypes

    import torch
    import torch.distributed as dist

    lib = _dev.load_library()
    dev = _dev.require_device()
    torch.cuda.set_device(dev)
    rank = dist.get_rank(group)
    nbytes = 8 + 4 * total  # the uint64 key (8-byte aligned), then int32 max|W| per component
    handle = ctypes.create_string_buffer(64)
    base = ctypes.c_void_p()
    if rank == 0:
        _dev.check(lib.sbw_ipc_alloc(nbytes, ctypes.byref(base), handle))
    obj = [handle.raw if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    if rank != 0:
        _dev.check(lib.sbw_ipc_open(ctypes.create_string_buffer(obj[0], 64), ctypes.byref(base)))
    root = int(base.value)
    try:
        stream = _dev.stream_handle(dev)
        if hi > lo:
            tab = _dev.device_table(s, dev)
            key = torch.zeros(1, dtype=torch.int64, device=dev)
            sb = lib.sbw_nl_scratch_bytes(s.n, s.m, lo, hi)
            scratch = torch.empty(max(1, sb), dtype=torch.uint8, device=dev)
            _dev.check(lib.sbw_nl(_dev.ptr(tab), _dev.table_bytes(s.m), s.n, s.m, lo, hi,
                                  root + 8 + 4 * (lo - 1), _dev.ptr(key), _dev.ptr(scratch), sb, stream))
            _dev.check(lib.sbw_key_merge(_dev.ptr(key), root, stream))
        torch.cuda.synchronize(dev)
        dist.barrier(group=group)  # every shard is in rank 0's memory
        out = torch.empty(2 + total, dtype=torch.int32, device=dev)
        _dev.check(lib.sbw_peer_copy(_dev.ptr(out), root, nbytes if return_values else 8, stream))
        torch.cuda.synchronize(dev)
        k = int(out[:2].view(torch.int64).item())
        values = maxabs_to_nl(out[2:], s.n) if return_values else None
        dist.barrier(group=group)  # nobody reads rank 0's buffer any more
    finally:
        if rank == 0:
            lib.sbw_ipc_free(base)
        else:
            lib.sbw_ipc_close(base)
    return k, values


def evaluate_distributed(s: SBox, group=None, compute=None, return_values: bool = True,
                         transport: str = "collective") -> tuple[NonlinearityResult, ColumnMaxima | None]:
    """Whole-S-box NL with the masks sharded over the ranks of `group`.

    Rank r owns partition_columns(2^m - 1, world)[r] (the reference's static
    partition, parallel.py:38-57).  Exchange: one all-reduce(MAX) of the
    packed (max|W| << 32 | ~v) key and, if `return_values`, one all-gather of
    the padded per-component NL shards.  `compute(s, lo, hi) -> (nl_int64,
    key)` defaults to the GPU; tests inject the CPU oracle to exercise the
    exchange on gloo.

    transport="p2p" (one process per GPU, CUDA devices required): no
    collective on the data path -- the shards' maxima and keys are written
    into rank 0's device memory through CUDA IPC mappings (_evaluate_p2p).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    total = (1 << s.m) - 1
    part = partition_columns(total, world)
    ranges = list(part.ranges) + [(total + 1, total + 1)] * (world - len(part.ranges))
    lo, hi = ranges[rank]
    if transport == "p2p":
        if compute is not None:
            raise ValueError("transport='p2p' runs the shards on the GPU; compute= is not supported")
        k, values = _evaluate_p2p(s, group, lo, hi, total, return_values)
        mxw = k >> 32
        gap = (1 << s.n) - mxw
        if gap & 1:
            raise AssertionError("spectrum maximum has wrong parity")
        result = NonlinearityResult(gap >> 1, 0xFFFFFFFF - (k & 0xFFFFFFFF), "distributed")
        return result, (ColumnMaxima(s.n, s.m, values) if return_values else None)
    if transport != "collective":
        raise ValueError(f"transport must be 'collective' or 'p2p', got {transport!r}")
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    count = hi - lo
    flag = None
    if compute is None:
        # GPU shards: the per-component values and the key stay on the GPU
        # for the collectives (no host round trip); the odd-gap flag is read
        # once at the end
        gdev = _dev.require_device()
        if count > 0:
            nl_t, key_t = _gpu_shard(s, lo, hi)
            flag = nl_t[count:]
            nl_t = nl_t[:count]
        else:
            nl_t = torch.zeros(0, dtype=torch.int64, device=gdev)
            key_t = torch.zeros(1, dtype=torch.int64, device=gdev)
        nl_t, key_t = nl_t.to(dev), key_t.to(dev)
    else:
        if count > 0:
            nl, key = compute(s, lo, hi)
        else:
            nl, key = np.zeros(0, dtype=np.int64), 0
        key_t = torch.tensor([key], dtype=torch.int64, device=dev)
        nl_t = torch.from_numpy(np.asarray(nl, dtype=np.int64)).to(dev)
    dist.all_reduce(key_t, op=dist.ReduceOp.MAX, group=group)
    cm = None
    if return_values:
        width = max(h - l for l, h in ranges)
        buf = torch.full((width,), -1, dtype=torch.int64, device=dev)
        buf[:count] = nl_t
        parts = torch.empty((world, width), dtype=torch.int64, device=dev)
        if backend == "nccl":
            dist.all_gather_into_tensor(parts, buf, group=group)
        else:
            dist.all_gather(list(parts.unbind(0)), buf, group=group)
        gathered = parts.cpu().numpy()  # the one device -> host copy of the values
        values = np.empty(total, dtype=np.int64)
        for (l, h), p in zip(ranges, gathered):
            if h > l:
                values[l - 1:h - 1] = p[: h - l]
        cm = ColumnMaxima(s.n, s.m, values)
    if flag is not None:
        check_nl_flag(int(flag.item()))
    k = int(key_t.item())
    mxw = k >> 32
    v = 0xFFFFFFFF - (k & 0xFFFFFFFF)
    gap = (1 << s.n) - mxw
    if gap & 1:
        raise AssertionError("spectrum maximum has wrong parity")
    return NonlinearityResult(gap >> 1, v, "distributed"), cm


def _key_of_maxima(mx, v_lo: int):
    """(max|W| << 32) | (0xFFFFFFFF - v) of a shard's per-component maxima,
    v = the smallest mask reaching the maximum (the reference's first
    argmin, nonlinearity.py:44-49).  Device tensors stay on the device."""
    import torch

    if isinstance(mx, np.ndarray):
        i = int(np.argmax(mx))
        return (int(mx[i]) << 32) | (0xFFFFFFFF - (v_lo + i))
    i = torch.argmax(mx)  # first maximal index
    return (mx[i].to(torch.int64) << 32) | (0xFFFFFFFF - (v_lo + i))


def spectrum_distributed(s: SBox, group=None, layout: str = "mask", compute=None,
                         max_bytes: int | None = None):
    """Materialised Walsh spectrum, sharded over the ranks of `group`.

    Rank r computes and keeps only its mask range (lo, hi) =
    partition_columns(2^m - 1, world)[r] (parallel.py:38-57) on its own GPU,
    in the reference's row layout (layout="mask": int32 [hi - lo, 2^n],
    rows[v - lo][u] = W(u, v), walsh.py:174) or x-major (layout="x": int32
    [2^n, hi - lo], wt[u][v - lo], walsh.py:117-131).  The matrix is never
    gathered; the only exchange is one all-reduce(MAX) of the packed
    (max|W|, smallest v) key, so every rank also gets the global NL.

    Returns (shard, (lo, hi), NonlinearityResult): the shard is a device
    tensor (or, with an injected `compute(s, lo, hi, layout) -> (numpy
    shard, numpy int32 max|W|)`, used by the CPU tests, a CPU tensor).
    `max_bytes` bounds the shard like the reference's retain-mode budget
    (walsh.py:220-222).
    """
    import torch
    import torch.distributed as dist

    if layout not in ("mask", "x"):
        raise ValueError(f"layout must be 'mask' or 'x', got {layout!r}")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    total = (1 << s.m) - 1
    ranges = list(partition_columns(total, world).ranges)
    ranges += [(total + 1, total + 1)] * (world - len(ranges))
    lo, hi = ranges[rank]
    count = hi - lo
    check_budget(count * (1 << s.n) * 4, max_bytes)
    backend = dist.get_backend(group)
    shape = (count, 1 << s.n) if layout == "mask" else (1 << s.n, count)
    if compute is None:
        dev = _dev.require_device()
        if count > 0:
            shard, mx = spectrum_device(s, lo, hi, layout=layout, device=dev)
            key_t = _key_of_maxima(mx, lo).reshape(1)
        else:
            shard = torch.empty(shape, dtype=torch.int32, device=dev)
            key_t = torch.zeros(1, dtype=torch.int64, device=dev)
    else:
        if count > 0:
            sh, mx = compute(s, lo, hi, layout)
            shard = torch.from_numpy(np.ascontiguousarray(sh, dtype=np.int32))
            key_t = torch.tensor([_key_of_maxima(np.asarray(mx), lo)], dtype=torch.int64)
        else:
            shard = torch.empty(shape, dtype=torch.int32)
            key_t = torch.zeros(1, dtype=torch.int64)
    red = key_t if backend == "nccl" else key_t.cpu()
    dist.all_reduce(red, op=dist.ReduceOp.MAX, group=group)
    k = int(red.item())
    mxw = k >> 32
    gap = (1 << s.n) - mxw
    if gap & 1:
        raise AssertionError("spectrum maximum has wrong parity")
    return shard, (lo, hi), NonlinearityResult(gap >> 1, 0xFFFFFFFF - (k & 0xFFFFFFFF), "distributed")
