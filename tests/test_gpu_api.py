"""GPU tests of the round-2 API surface: every reference name on the hot path
exists, runs on libsbw, and matches the reference's own outputs.

  fwht_column_in_place on every integer dtype + strided/negative views
                             (walsh.py:73-104)   -> sbw_fwht_inplace_strided
  column_nonlinearity        (walsh.py:107-114)
  build_polarity_xmajor      (walsh.py:117-131)  -> sbw_polarity layout 1
  transform_xmajor_in_place  (walsh.py:134-137)  -> sbw_fwht_inplace_strided
  transform_rows_in_place on non-int32 stores (walsh.py:140-152)
  submodule imports the reference's own tests use (sboxeval.walsh, .parallel,
  .nonlinearity, .memory, .bench, .sbox, .cli)
  multi-GPU fwht_parallel (parallel.py:64-133), bench.py --gpus N spawning

Goldens: tests/golden/golden_api.{json,npz} (make_golden_api.py ran the
reference); the oracle restatement (oracle/sbw_oracle.py) is pinned to them
in tests/test_oracle.py and checks the larger cases here.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1912_03732_b200 as sw
from oracle import sbw_oracle as orc
from tests.util import sha

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


@pytest.fixture(scope="module")
def api():
    with open(os.path.join(HERE, "golden", "golden_api.json")) as f:
        meta = json.load(f)
    with np.load(os.path.join(HERE, "golden", "golden_api.npz")) as z:
        arrays = {k: z[k] for k in z.files}
    return meta, arrays


def test_typed_columns_match_reference(api):
    meta, arrays = api
    for rec in meta["columns"]:
        col = arrays[rec["key"] + "_in"].copy()
        out, mx = sw.fwht_column_in_place(col)
        assert out is col and col.dtype == arrays[rec["key"] + "_in"].dtype
        assert np.array_equal(col, arrays[rec["key"] + "_out"]), rec
        assert mx == rec["max_abs"] and type(mx) is int, (rec, mx)


def test_strided_and_negative_views_match_reference(api):
    meta, arrays = api
    base = arrays["strided_base_in"].copy()
    _, mx = sw.fwht_column_in_place(base[::3])
    assert np.array_equal(base, arrays["strided_base_out"]) and mx == meta["strided_max_abs"]
    neg = arrays["neg_in"].copy()
    _, mx = sw.fwht_column_in_place(neg[::-1])
    assert np.array_equal(neg, arrays["neg_out"]) and mx == meta["neg_max_abs"]


@pytest.mark.parametrize("dtype", ["int8", "uint16", "int64", "uint64"])
@pytest.mark.parametrize("k", [12, 17])
def test_typed_long_columns_against_oracle(dtype, k):
    info = np.iinfo(dtype)
    col = np.random.default_rng(k).integers(info.min, info.max, size=1 << k, dtype=dtype,
                                            endpoint=True)
    want, wmx = orc.fwht_column_typed(col)
    got = col.copy()
    _, mx = sw.fwht_column_in_place(got)
    assert np.array_equal(got, want) and mx == wmx


def test_read_only_and_non_integer_columns_raise():
    ro = np.ones(8, dtype=np.int32)
    ro.flags.writeable = False
    with pytest.raises(ValueError, match="read-only"):
        sw.fwht_column_in_place(ro)
    with pytest.raises(TypeError):
        sw.fwht_column_in_place(np.ones(8, dtype=np.float64))
    with pytest.raises(ValueError, match="power of two"):
        sw.fwht_column_in_place(np.ones(12, dtype=np.int16))


def test_transform_rows_in_place_other_dtypes(api):
    meta, arrays = api
    for rec in meta["rows"]:
        dt = rec["dtype"]
        rows = arrays[f"rows_{dt}_in"].copy()
        mo = np.zeros(rows.shape[0], dtype=np.int64)
        sw.transform_rows_in_place(rows, maxima_out=mo)
        assert rows.dtype == np.dtype(dt)
        assert np.array_equal(rows, arrays[f"rows_{dt}_out"])
        assert np.array_equal(mo, arrays[f"rows_{dt}_maxima"])


def test_column_nonlinearity(api):
    meta, _ = api
    for pw, mx, nl in meta["column_nonlinearity"]:
        assert sw.column_nonlinearity(pw, mx) == nl
        assert sw.walsh.column_nonlinearity(pw, mx) == nl
    with pytest.raises(AssertionError, match="odd"):
        sw.column_nonlinearity(256, 31)


def test_build_polarity_xmajor_and_transform(api):
    meta, _ = api
    for rec in meta["xmajor"]:
        s = sw.generate_sbox(rec["n"], rec["m"], rec["seed"], bijective=rec["bijective"])
        wt = sw.build_polarity_xmajor(s)
        assert wt.shape == (1 << s.n, (1 << s.m) - 1) and wt.dtype == np.int32
        assert sha(wt) == rec["sha_polarity_xmajor"]
        assert sw.transform_xmajor_in_place(wt) is None
        assert sha(wt) == rec["sha_spectrum_xmajor"]
    with pytest.raises(sw.MemoryBudgetError):
        sw.build_polarity_xmajor(sw.generate_sbox(8, 8, 1), max_bytes=1000)


@pytest.mark.parametrize("n,m", [(13, 6), (14, 5), (16, 4), (17, 3), (18, 2)])
def test_xmajor_store_transform_against_oracle(n, m):
    """x-major stores above n = 12: the strided device butterfly over the
    reference's wt[x][v-1] layout, against the oracle's mask-major spectrum."""
    s = sw.generate_sbox(n, m, seed=n)
    wt = sw.build_polarity_xmajor(s)
    assert np.array_equal(wt, orc.polarity_block(s.table, 1, 1 << m).T)
    sw.transform_xmajor_in_place(wt)
    assert np.array_equal(wt, orc.spectrum(s.table, n, 1, 1 << m).T)


def test_transform_xmajor_int16_wraps_like_numpy():
    wt = np.random.default_rng(5).integers(-30000, 30000, size=(1 << 9, 37)).astype(np.int16)
    want = orc.xmajor_spectrum_typed(wt)
    got = wt.copy()
    sw.transform_xmajor_in_place(got)
    assert np.array_equal(got, want)
    sw.transform_xmajor_in_place(np.zeros((8, 0), dtype=np.int32))  # no columns: no-op
    with pytest.raises(ValueError, match="power of two"):
        sw.transform_xmajor_in_place(np.zeros((6, 3), dtype=np.int32))


def test_reference_submodules_resolve():
    """The import paths the reference's own suite uses (pkg/tests/*.py)."""
    import importlib

    for mod, names in {
        "walsh": ["WalshSpectrum", "ColumnMaxima", "fwht_column_in_place", "column_nonlinearity",
                  "build_polarity_xmajor", "transform_xmajor_in_place", "transform_rows_in_place",
                  "fwht_rowmajor", "fwht_transposed", "fwht_fused", "walsh_direct", "write_spectrum"],
        "parallel": ["ColumnPartition", "partition_columns", "default_workers", "fwht_parallel"],
        "nonlinearity": ["METHODS", "NonlinearityResult", "SizeCapError", "evaluate",
                         "nonlinearity_bruteforce", "nonlinearity_from_maxima",
                         "nonlinearity_from_spectrum"],
        "memory": ["MemoryBudgetError", "AllocationTracker", "spectrum_allocations", "check_budget",
                   "default_budget", "physical_memory_bytes"],
        "bench": ["BenchRecord", "BenchVerificationError", "SpeedupRow", "run_benchmark",
                  "speedup_report", "write_csv", "read_csv", "nonlinearity_bruteforce"],
        "sbox": ["SBox", "SBoxFormatError", "PolarityTruthTable", "AES_SBOX", "aes_sbox",
                 "identity_sbox", "generate_sbox", "component_value", "polarity_row",
                 "polarity_truth_table", "memory_estimate", "parse_sbox", "render_sbox"],
        "cli": ["main"],
    }.items():
        m = importlib.import_module(f"paper_1912_03732_b200.{mod}")
        for name in names:
            assert hasattr(m, name), (mod, name)


def test_fwht_parallel_across_all_gpus():
    """Shards mapped round-robin over every visible GPU (parallel.py:64-133
    contract: bit-identical for any worker count)."""
    import torch

    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        pytest.skip("needs >= 2 GPUs")
    s = sw.generate_sbox(16, 16, 0, bijective=True)
    g = np.load(os.path.join(HERE, "golden", "golden_arrays.npz"))["maxima_16x16"]
    for workers in (ngpu, 2 * ngpu + 1):
        _, cm = sw.fwht_parallel(s, workers=workers, mode="stream")
        assert np.array_equal(cm.values, g)
    small = sw.generate_sbox(10, 9, 3)
    spec, cm = sw.fwht_parallel(small, workers=ngpu, mode="retain")
    assert np.array_equal(spec.rows, orc.spectrum(small.table, 10, 1, 512))
    assert torch.cuda.current_device() == 0


def test_calls_run_on_the_buffers_device_not_the_current_one():
    """libsbw picks the device from the stream / data pointer (include/sbw.h):
    a call made while another device is current still runs where its buffers
    live and leaves the current device unchanged."""
    import torch

    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        pytest.skip("needs >= 2 GPUs")
    s = sw.generate_sbox(12, 12, 0, bijective=True)
    torch.cuda.set_device(0)
    mx, key = sw.component_max_abs_device(s, device="cuda:1")
    assert mx.device.index == 1 and torch.cuda.current_device() == 0
    assert np.array_equal(mx.cpu().numpy(), orc.component_max_abs(s.table, 12, 1, 4096))


def test_bench_spawns_ranks_without_torchrun():
    """`python bench.py --gpus 2` (no torchrun) starts two ranks itself and
    prints one rank-0 line with n_gpus 2.  One GPU here: the gloo plumbing
    backend lets both ranks share it (timings meaningless, plumbing only)."""
    env = dict(os.environ, SBW_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
                        "--warmup", "3", "--config", "12x12", "--no-cpu"],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert (line["result"]["nl"], line["result"]["argmin_v"]) == (1872, 3572)


def test_libsbw_calls_capture_into_a_cuda_graph():
    """libsbw entry points are stream-ordered and capturable: a 12x12 NL
    captured into a CUDA graph replays to the reference's maxima (the device
    selection must not query the capturing stream's device)."""
    import torch

    import paper_1912_03732_b200.device as d

    s = sw.generate_sbox(12, 12, 0, bijective=True)
    lib = d.load_library()
    dev = torch.device("cuda", 0)
    tab = d.device_table(s, dev)
    mx = torch.empty(4095, dtype=torch.int32, device=dev)
    key = torch.zeros(1, dtype=torch.int64, device=dev)
    sb = lib.sbw_nl_scratch_bytes(12, 12, 1, 4096)
    scratch = torch.empty(max(1, sb), dtype=torch.uint8, device=dev)
    st = torch.cuda.Stream(dev)

    def call():
        d.check(lib.sbw_nl(tab.data_ptr(), 2, 12, 12, 1, 4096, mx.data_ptr(), key.data_ptr(),
                           scratch.data_ptr(), sb, st.cuda_stream))

    with torch.cuda.stream(st):
        call()  # first call: per-device setup outside the capture
    st.synchronize()
    mx.zero_()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st, capture_error_mode="relaxed"):
        call()
    graph.replay()
    torch.cuda.synchronize()
    assert np.array_equal(mx.cpu().numpy().astype(np.int64), orc.component_max_abs(s.table, 12, 1, 4096))
