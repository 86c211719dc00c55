"""GPU parity: libsbw kernels vs the pinned oracle and the reference goldens.

Bit-exact everywhere (integer work).  Mirrors the reference's own suite:
pkg/tests/test_walsh.py, test_nonlinearity.py, test_parallel.py,
test_acceptance.py (known answers, 250-box equivalence, Parseval,
determinism across worker counts, stream accounting).
"""
import os

import numpy as np
import pytest

import paper_1912_03732_b200 as sw
from oracle import sbw_oracle as orc
from tests.util import sha

pytestmark = pytest.mark.gpu

CFG = {"8x8": (8, 8, True), "12x12": (12, 12, True), "16x16": (16, 16, True),
       "20x20": (20, 20, False), "24x16": (24, 16, False)}


def box(name):
    n, m, bij = CFG[name]
    return sw.generate_sbox(n, m, 0, bijective=bij)


def test_native_library_is_loaded():
    import paper_1912_03732_b200.device as d

    d.load_library()
    before = d.launch_count()
    sw.fwht_fused(sw.aes_sbox(), mode="stream")
    assert d.launch_count() > before


# ---------------------------------------------------------------- AES -------
def test_aes_everything(golden):
    aes = sw.aes_sbox()
    g = golden["aes"]
    spec, cm = sw.fwht_fused(aes, mode="retain")
    assert sha(spec.rows) == g["sha_mask_major"]
    assert sha(cm.values) == g["sha_maxima_i64"]
    assert np.all(cm.values == 112)
    _, cm2 = sw.fwht_fused(aes, mode="stream")
    assert np.array_equal(cm.values, cm2.values)
    xm, _ = sw.spectrum_device(aes, layout="x")
    assert sha(xm.cpu().numpy()) == g["sha_x_major"]
    assert sha(sw.fwht_rowmajor(aes).rows) == g["sha_mask_major"]
    assert sha(sw.fwht_transposed(aes).rows) == g["sha_mask_major"]
    for method in sw.METHODS:
        for workers in (None, 1, 2, 4, 10):
            r = sw.evaluate(aes, method=method, workers=workers)
            assert r.value == 112 and r.method == method
            if method != "bruteforce":
                assert r.argmin_v == 1


def test_aes_exhaustive_direct_max_is_32():
    aes = sw.aes_sbox()
    u, v = np.meshgrid(np.arange(256), np.arange(1, 256))
    w = sw.walsh_direct_many(aes, u.ravel(), v.ravel())
    assert int(np.abs(w).max()) == 32
    rows = sw.fwht_transposed(aes).rows
    assert np.array_equal(w.reshape(255, 256), rows)


# ------------------------------------------------------- BASELINE configs ---
@pytest.mark.parametrize("name", ["8x8", "12x12"])
def test_materialised_configs(golden, name):
    s = box(name)
    g = golden["configs"][name]
    assert sha(s.table) == g["sha_table_u32"]
    spec, cm = sw.fwht_fused(s, mode="retain")
    assert sha(spec.rows) == g["sha_mask_major"]
    assert sha(cm.values) == g["sha_maxima_i64"]
    assert sha(sw.fwht_transposed(s).rows) == g["sha_mask_major"]
    assert sha(sw.fwht_rowmajor(s).rows) == g["sha_mask_major"]
    xm, mx = sw.spectrum_device(s, layout="x")
    assert sha(xm.cpu().numpy()) == g["sha_x_major"]
    _, cms = sw.fwht_fused(s, mode="stream")
    assert np.array_equal(cms.values, cm.values)
    r = sw.nonlinearity_from_spectrum(spec)
    assert (r.value, r.argmin_v) == (g["nl"], g["argmin_v"])
    r = sw.nonlinearity_from_maxima(cms)
    assert (r.value, r.argmin_v) == (g["nl"], g["argmin_v"])


def test_16x16_full_fused_nl(golden, golden_arrays):
    s = box("16x16")
    _, cm = sw.fwht_fused(s, mode="stream")
    assert np.array_equal(cm.values, golden_arrays["maxima_16x16"])
    assert sha(cm.values) == golden["configs"]["16x16"]["sha_maxima_i64"]
    r = sw.nonlinearity_from_maxima(cm)
    assert (r.value, r.argmin_v) == (31942, 44828)
    mx, key = sw.component_max_abs_device(s)
    assert sw.walsh.decode_key(key, 16) == (31942, 44828, 1652)


def test_16x16_materialised_slices():
    s = box("16x16")
    for lo, hi in [(1, 33), (44820, 44836), (65504, 65536)]:
        rows, mx = sw.spectrum_device(s, lo, hi)
        want = orc.spectrum(s.table, 16, lo, hi)
        assert np.array_equal(rows.cpu().numpy(), want)
        assert np.array_equal(mx.cpu().numpy(), np.abs(want).max(axis=1))
    rows, _ = sw.spectrum_device(s, 1, 2)
    assert rows[0, :8].cpu().tolist() == [0, -368, 440, 104, 52, 348, 260, -196]


@pytest.mark.parametrize("name,masks", [("20x20", 9), ("24x16", 9)])
def test_large_configs_subset(golden, name, masks):
    s = box(name)
    n, m = s.n, s.m
    sub = golden["configs"][name]["subset"]
    for rec in sub:
        v = rec["v"]
        mx, key = sw.component_max_abs_device(s, v, v + 1)
        assert int(mx[0]) == rec["max_abs"], rec
    mx, _ = sw.component_max_abs_device(s, 1, 9)
    assert mx.cpu().tolist() == [r["max_abs"] for r in sub if r["v"] <= 8]
    rows, _ = sw.spectrum_device(s, 1, 2)
    r0 = rows[0].cpu().numpy()
    assert r0[:8].tolist() == sub[0]["w_head"]
    assert int(np.argmax(np.abs(r0.astype(np.int64)))) == sub[0]["argmax_u"]


def test_20x20_materialised_vs_oracle():
    s = box("20x20")
    for v in (3, 777777):
        rows, mx = sw.spectrum_device(s, v, v + 1)
        want = orc.spectrum(s.table, 20, v, v + 1)
        assert np.array_equal(rows.cpu().numpy(), want)


@pytest.mark.slow
def test_20x20_full_nl_consistency():
    """Full 2^20 - 1 components: the fused range result equals per-shard
    results (any partition) and sampled masks equal the oracle."""
    s = box("20x20")
    mx, key = sw.component_max_abs_device(s)
    full = mx.cpu().numpy()
    nl, v, mw = sw.walsh.decode_key(key, 20)
    assert mw == full.max() and v == int(np.argmax(full)) + 1
    rng = np.random.default_rng(5)
    for vv in rng.integers(1, 1 << 20, size=4):
        vv = int(vv)
        want = orc.component_max_abs(s.table, 20, vv, vv + 1)
        assert full[vv - 1] == want[0]
    a, _ = sw.component_max_abs_device(s, 1, 300001)
    b, _ = sw.component_max_abs_device(s, 300001, 1 << 20)
    assert np.array_equal(np.concatenate([a.cpu().numpy(), b.cpu().numpy()]), full)


# ----------------------------------------------- shapes n, m = 1..24 --------
SHAPES = [(n, m) for n in range(1, 17) for m in (1, 2, 5, 9)] + [(3, 24), (5, 20), (8, 17), (16, 17)]


@pytest.mark.parametrize("n,m", SHAPES)
def test_every_shape_fused_and_spectrum(n, m):
    s = sw.generate_sbox(n, m, seed=n * 31 + m)
    top = 1 << m
    ranges = [(1, top)] if top <= 4096 else [(1, 200), (top - 300, top), (top // 2, top // 2 + 7)]
    for lo, hi in ranges:
        mx, _ = sw.component_max_abs_device(s, lo, hi)
        want = orc.component_max_abs(s.table, n, lo, hi)
        assert np.array_equal(mx.cpu().numpy(), want), (n, m, lo, hi)
        if (hi - lo) << n <= (1 << 26):
            rows, mx2 = sw.spectrum_device(s, lo, hi)
            assert np.array_equal(rows.cpu().numpy(), orc.spectrum(s.table, n, lo, hi))
            assert np.array_equal(mx2.cpu().numpy(), want)


@pytest.mark.parametrize("n", [17, 18, 19, 21, 22, 23])
def test_multipass_shapes(n):
    m = 4
    s = sw.generate_sbox(n, m, seed=n)
    mx, key = sw.component_max_abs_device(s)
    want = orc.component_max_abs(s.table, n, 1, 16)
    assert np.array_equal(mx.cpu().numpy(), want)
    rows, _ = sw.spectrum_device(s, 5, 7)
    assert np.array_equal(rows.cpu().numpy(), orc.spectrum(s.table, n, 5, 7))


def test_identity_16_full_range_stress():
    # every component is linear: |W| = 2^16 exactly at one u
    s = sw.identity_sbox(16)
    _, cm = sw.fwht_fused(s, mode="stream")
    assert np.all(cm.values == 0)
    rows, mx = sw.spectrum_device(s, 1, 64)
    assert np.all(mx.cpu().numpy() == 1 << 16)
    assert np.array_equal(rows.cpu().numpy(), orc.spectrum(s.table, 16, 1, 64))


def test_partially_affine_16():
    """Components that are affine (|W| = 2^16, the packed-lane wrap case) next
    to random ones in the same box."""
    rng = np.random.default_rng(11)
    t = (np.arange(1 << 16, dtype=np.uint32) & 0xFF) | (rng.integers(0, 256, 1 << 16,
                                                                    dtype=np.uint32) << 8)
    s = sw.SBox(16, 16, t)
    for lo, hi in [(1, 300), (250, 262), (65400, 65536)]:
        mx, _ = sw.component_max_abs_device(s, lo, hi)
        assert np.array_equal(mx.cpu().numpy(), orc.component_max_abs(s.table, 16, lo, hi))
    mx, key = sw.component_max_abs_device(s)
    assert np.all(mx.cpu().numpy()[:255] == 1 << 16)
    assert sw.walsh.decode_key(key, 16)[:2] == (0, 1)


def test_identity_and_constant_24_bit():
    s = sw.SBox(17, 3, np.zeros(1 << 17, dtype=np.uint32))
    mx, key = sw.component_max_abs_device(s)
    assert np.all(mx.cpu().numpy() == 1 << 17)  # W(0, v) = 2^n for every v
    s = sw.SBox(18, 18, np.arange(1 << 18, dtype=np.uint32))
    mx, _ = sw.component_max_abs_device(s, 1, 40)
    assert np.all(mx.cpu().numpy() == 1 << 18)


# --------------------------------------------- reference suite equivalents --
def test_small_sweep_against_reference_goldens(golden):
    for rec in golden["small"]["sweep"]:
        s = sw.generate_sbox(rec["n"], rec["m"], rec["seed"], rec["bijective"])
        spec, cm = sw.fwht_fused(s, mode="retain")
        assert sha(spec.rows) == rec["sha_mask_major"], rec
        assert sha(cm.values) == rec["sha_maxima_i64"], rec
        r = sw.nonlinearity_from_maxima(cm)
        assert (r.value, r.argmin_v) == (rec["nl"], rec["argmin_v"])
        if "nl_bruteforce" in rec:
            assert sw.nonlinearity_bruteforce(s).value == rec["nl_bruteforce"]


def test_specials(golden):
    for rec in golden["small"]["specials"]:
        if rec["table"] is not None:
            s = sw.SBox(rec["n"], rec["m"], np.array(rec["table"], dtype=np.uint32))
        else:
            s = sw.identity_sbox(rec["n"])
        spec, cm = sw.fwht_fused(s, mode="retain")
        assert sha(spec.rows) == rec["sha_mask_major"], rec["label"]
        r = sw.nonlinearity_from_maxima(cm)
        assert (r.value, r.argmin_v) == (rec["nl"], rec["argmin_v"])


def test_oracle_equivalence_sweep_250():
    for n, m in [(3, 3), (4, 4), (5, 5), (6, 4), (4, 6)]:
        for seed in range(50):
            s = sw.generate_sbox(n, m, seed)
            rows = sw.fwht_transposed(s).rows
            assert np.array_equal(rows, orc.spectrum(s.table, n, 1, 1 << m))
            assert np.array_equal(sw.fwht_rowmajor(s).rows, rows)
            vals = {sw.nonlinearity_from_spectrum(sw.WalshSpectrum(n, m, rows)).value,
                    sw.evaluate(s, method="fused").value,
                    sw.nonlinearity_bruteforce(s).value}
            assert len(vals) == 1


def test_parseval_suite():
    sizes = [(4, 4), (5, 7), (6, 6), (7, 3), (3, 8), (8, 8), (9, 5), (5, 9), (10, 10), (7, 7)]
    for seed in range(20):
        n, m = sizes[seed % len(sizes)]
        spec, _ = sw.fwht_fused(sw.generate_sbox(n, m, seed), mode="retain")
        sums = np.sum(spec.rows.astype(np.int64) ** 2, axis=1)
        assert np.all(sums == np.int64(1) << (2 * n))
        assert np.all(spec.rows % 2 == 0)


@pytest.mark.slow
def test_16x16_materialised_parseval_full():
    """Full 16 GiB spectrum on the device: Parseval per row and maxima equal
    the fused path (size-independent properties at the full config)."""
    import torch

    s = box("16x16")
    rows, mx = sw.spectrum_device(s)
    mx_f, _ = sw.component_max_abs_device(s)
    assert torch.equal(mx, mx_f)
    for a in range(0, rows.shape[0], 4096):
        blk = rows[a:a + 4096].to(torch.int64)
        assert bool(((blk * blk).sum(dim=1) == (1 << 32)).all())
    del rows


def test_thread_determinism_workers_1_to_12():
    s = sw.generate_sbox(10, 10, seed=2024)
    ref_spec, ref_cm = sw.fwht_parallel(s, workers=1, mode="retain")
    for w in range(2, 13):
        spec, cm = sw.fwht_parallel(s, workers=w, mode="retain")
        assert np.array_equal(spec.rows, ref_spec.rows)
        assert np.array_equal(cm.values, ref_cm.values)
        _, cms = sw.fwht_parallel(s, workers=w, mode="stream")
        assert np.array_equal(cms.values, ref_cm.values)


def test_stream_accounting():
    s = sw.generate_sbox(10, 10, seed=12)
    sw.spectrum_allocations.reset_peak()
    sw.fwht_parallel(s, workers=4, mode="stream")
    assert sw.spectrum_allocations.peak_bytes <= 4 * (1 << 10) * 4
    assert sw.spectrum_allocations.current_bytes == 0
    sw.fwht_fused(s, mode="retain")
    assert sw.spectrum_allocations.current_bytes == 0


def test_budget_errors_and_modes():
    s = sw.generate_sbox(8, 8, seed=3)
    with pytest.raises(sw.MemoryBudgetError):
        sw.fwht_rowmajor(s, max_bytes=1024)
    with pytest.raises(sw.MemoryBudgetError):
        sw.fwht_fused(s, mode="retain", max_bytes=1024)
    with pytest.raises(sw.MemoryBudgetError):
        sw.fwht_parallel(s, workers=2, mode="retain", max_bytes=4096)
    with pytest.raises(ValueError, match="retain.*stream"):
        sw.fwht_fused(sw.identity_sbox(2), mode="drop")


# ------------------------------------------------------- column kernel ------
def test_columns_against_reference_goldens(golden, golden_arrays):
    for rec in golden["small"]["columns"]:
        key = "col_in_wrap" if rec.get("label") == "wrap" else f"col_in_{rec['k']}"
        col = golden_arrays[key].copy()
        out, mx = sw.fwht_column_in_place(col)
        assert out is col
        assert sha(col) == rec["sha_out"] and mx == rec["max_abs"], rec


def test_column_kernel_cases():
    col = np.array([1, 1, 1, -1], dtype=np.int32)
    _, mx = sw.fwht_column_in_place(col)
    assert col.tolist() == [2, 2, 2, -2] and mx == 2
    for n in (1, 2, 3, 6):
        col = np.ones(1 << n, dtype=np.int32)
        _, mx = sw.fwht_column_in_place(col)
        assert col[0] == 1 << n and np.all(col[1:] == 0) and mx == 1 << n
    for k in range(1, 13):
        orig = np.random.default_rng(k).choice([-1, 1], size=1 << k).astype(np.int32)
        col = orig.copy()
        sw.fwht_column_in_place(col)
        sw.fwht_column_in_place(col)
        assert np.array_equal(col, (1 << k) * orig)
    mat = np.zeros((4, 3), dtype=np.int32)
    mat[:, 1] = [1, 1, 1, -1]
    sw.fwht_column_in_place(mat[:, 1])
    assert mat[:, 1].tolist() == [2, 2, 2, -2] and np.all(mat[:, [0, 2]] == 0)
    col = np.array([-7], dtype=np.int32)
    _, mx = sw.fwht_column_in_place(col)
    assert col[0] == -7 and mx == 7
    with pytest.raises(ValueError, match="power of two"):
        sw.fwht_column_in_place(np.ones(6, dtype=np.int32))


@pytest.mark.parametrize("k", [13, 17, 20, 24])
def test_long_columns(k):
    rng = np.random.default_rng(k)
    vals = rng.integers(-5, 6, size=1 << k).astype(np.int32)
    want, wmx = orc.fwht_column(vals)
    col = vals.copy()
    _, mx = sw.fwht_column_in_place(col)
    assert np.array_equal(col, want) and mx == wmx


@pytest.mark.parametrize("rows_n,k", [(3, 12), (5, 13), (2, 16), (1, 18)])
def test_rows_in_place_tile_pass(rows_n, k):
    """k >= 12 takes the shared-memory 12-bit tile pass (k_inplace_tile12) first;
    values up to 2^30 exercise int32 wrap-around in every phase."""
    rng = np.random.default_rng(100 + k)
    rows = rng.integers(-(1 << 30), 1 << 30, size=(rows_n, 1 << k)).astype(np.int32)
    rows[0, :] = rng.integers(-5, 6, size=1 << k)
    want = np.stack([orc.fwht_column(r)[0] for r in rows])
    wmx = [orc.fwht_column(r)[1] for r in rows]
    got = rows.copy()
    for i in range(rows_n):
        _, mx = sw.fwht_column_in_place(got[i])
        assert mx == wmx[i], (i, mx, wmx[i])
    assert np.array_equal(got, want)
    # all rows at once (one launch, per-row maxima)
    got2 = rows.copy()
    mx_rows = sw.walsh._inplace_rows(got2)
    assert np.array_equal(got2, want) and mx_rows.tolist() == wmx


def test_transform_rows_in_place_with_maxima():
    s = sw.generate_sbox(9, 6, seed=4)
    rows = orc.polarity_block(s.table, 1, 64)
    out = np.zeros(63, dtype=np.int64)
    sw.transform_rows_in_place(rows, maxima_out=out)
    assert np.array_equal(rows, orc.spectrum(s.table, 9, 1, 64))
    assert np.array_equal(out, orc.component_nl(s.table, 9, 1, 64))
    bad = np.ones((2, 4), dtype=np.int32)
    bad[1, 0] = 2  # sum 5 at u = 0: odd gap
    with pytest.raises(AssertionError):
        sw.transform_rows_in_place(bad, maxima_out=np.zeros(2, dtype=np.int64))


# ------------------------------------------------------ polarity / misc -----
def test_polarity_tables():
    s = sw.generate_sbox(7, 6, seed=8)
    ptt = sw.polarity_truth_table(s)
    assert np.array_equal(ptt.rows, orc.polarity_block(s.table, 1, 64))
    assert np.array_equal(sw.polarity_row(s, 0), np.ones(128, dtype=np.int32))
    buf = np.empty(128, dtype=np.int32)
    assert sw.polarity_row(s, 5, out=buf) is buf
    assert np.array_equal(buf, orc.polarity(s.table, 5))
    aes = sw.polarity_truth_table(sw.aes_sbox())
    assert aes.rows[0, 0] == -1 and aes.rows[0, 1] == 1
    with pytest.raises(sw.MemoryBudgetError):
        sw.polarity_truth_table(sw.generate_sbox(8, 8, seed=1), max_bytes=1000)


def test_walsh_direct_api():
    s = sw.generate_sbox(5, 5, seed=1)
    assert sw.walsh_direct(s, 0, 0) == 32
    for v in range(1, 32):
        for u in range(32):
            assert sw.walsh_direct(s, u, v) == orc.walsh_direct(s.table, 5, u, v)
    with pytest.raises(IndexError):
        sw.walsh_direct(sw.identity_sbox(3), 8, 0)
    with pytest.raises(IndexError):
        sw.walsh_direct(sw.identity_sbox(3), 0, 8)


def test_nonlinearity_properties():
    for n, seed in [(4, 1), (4, 2), (6, 3), (6, 4)]:
        r = sw.evaluate(sw.generate_sbox(n, n, seed), method="fused")
        assert r.value <= (1 << (n - 1)) - (1 << (n // 2 - 1))
    r = sw.nonlinearity_from_maxima(sw.fwht_fused(sw.identity_sbox(4))[1])
    assert (r.value, r.argmin_v) == (0, 1)
    with pytest.raises(sw.SizeCapError):
        sw.nonlinearity_bruteforce(sw.generate_sbox(9, 9, seed=0))
    with pytest.raises(ValueError, match="unknown method"):
        sw.evaluate(sw.identity_sbox(2), method="magic")


def test_sbw_nl_host_entry_point():
    """The host-buffer C entry point a plugin binding would call."""
    import ctypes

    import paper_1912_03732_b200.device as d

    s = box("12x12")
    nl = np.empty(4095, dtype=np.int64)
    out3 = np.empty(3, dtype=np.int64)
    d.check(d.load_library().sbw_nl_host(s.table.ctypes.data, 12, 12, 1, 4096,
                                         nl.ctypes.data, out3.ctypes.data, 0))
    assert out3.tolist() == [1872, 3572, 352]
    assert np.array_equal(nl, orc.component_nl(s.table, 12, 1, 4096))
    del ctypes


@pytest.mark.parametrize("pin_table,pin_nl", [(True, True), (True, False), (False, True)])
def test_sbw_nl_host_page_locked_buffers(pin_table, pin_nl):
    """Page-locked caller buffers take the direct-DMA branch of sbw_nl_host
    (uint32 table straight to the device, NL straight into the caller's array)."""
    import torch

    import paper_1912_03732_b200.device as d

    s = box("16x16")
    table = np.ascontiguousarray(s.table)
    nl = np.zeros(65535, dtype=np.int64)
    out3 = np.empty(3, dtype=np.int64)
    cudart = torch.cuda.cudart()
    regs = [a for a, p in ((table, pin_table), (nl, pin_nl)) if p]
    for a in regs:
        assert int(cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)) == 0
    try:
        d.check(d.load_library().sbw_nl_host(table.ctypes.data, 16, 16, 1, 65536, nl.ctypes.data,
                                             out3.ctypes.data, 0))
    finally:
        for a in regs:
            cudart.cudaHostUnregister(a.ctypes.data)
    assert out3.tolist() == [31942, 44828, 1652]
    # the reference's ColumnMaxima.values for 16x16 are the per-component NLs
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_arrays.npz"))["maxima_16x16"]
    assert np.array_equal(nl, g.astype(np.int64))


def test_distributed_single_rank_nccl():
    import os

    import torch
    import torch.distributed as dist

    if dist.is_initialized():
        pytest.skip("process group already initialised")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        s = box("12x12")
        r, cm = sw.evaluate_distributed(s)
        assert (r.value, r.argmin_v) == (1872, 3572)
        assert np.array_equal(cm.values, orc.component_nl(s.table, 12, 1, 4096))
    finally:
        dist.destroy_process_group()
    del torch


# ---------------------------------------------- CLI + bench harness (GPU) ----
def _boxfile(tmp_path, name, s):
    p = tmp_path / name
    p.write_text(sw.render_sbox(s))
    return str(p)


def test_cli_nl_walsh_verify(tmp_path, capsys):
    from paper_1912_03732_b200.cli import main

    aes = _boxfile(tmp_path, "aes.sbox", sw.aes_sbox())
    assert main(["nl", aes]) == 0
    out = capsys.readouterr().out
    assert out.startswith("nl = 112") and "argmin v = 1" in out
    for method in ("fused", "bruteforce", "transposed"):
        assert main(["nl", aes, "--method", method]) == 0
        assert capsys.readouterr().out.startswith("nl = 112")
    r8 = _boxfile(tmp_path, "r8.sbox", sw.generate_sbox(8, 8, 1))
    assert main(["nl", r8, "--max-mem", str(8 * 256 * 4), "--mode", "stream",
                 "--workers", "2"]) == 0
    idf = _boxfile(tmp_path, "id2.sbox", sw.identity_sbox(2))
    wout = tmp_path / "id2.wspec"
    assert main(["walsh", idf, "--out", str(wout)]) == 0
    lines = wout.read_text().splitlines()
    assert lines[0] == "2 2" and len(lines) == 4
    for line in lines[1:]:
        assert sorted(map(abs, map(int, line.split()))) == [0, 0, 0, 4]
    r6 = _boxfile(tmp_path, "r6.sbox", sw.generate_sbox(6, 5, 3))
    assert main(["verify", r6, "--max-workers", "4"]) == 0
    assert capsys.readouterr().out.count("PASS") == 4
    assert main(["verify", r6, "--max-workers", "2", "--inject-corruption"]) == 5
    out = capsys.readouterr().out
    assert "FAIL direct-oracle equivalence" in out and "FAIL parseval" in out


def test_cli_bench_csv_and_harness(tmp_path, monkeypatch):
    import paper_1912_03732_b200.bench as h
    from paper_1912_03732_b200.cli import main

    path = _boxfile(tmp_path, "r7.sbox", sw.generate_sbox(7, 7, 2))
    out = tmp_path / "rep.csv"
    assert main(["bench", path, "--methods", "fused,transposed,parallel", "--workers", "1,3",
                 "--reps", "2", "--out", str(out)]) == 0
    rows = sw.read_csv(out.read_text())
    assert [(r["method"], r["workers"]) for r in rows] == [
        ("fused", 1), ("parallel", 1), ("parallel", 3), ("transposed", 1)]
    assert all(r["mean_ms"] > 0 and r["transform_only_mean_ms"] > 0 for r in rows)
    # verify-before-time: a wrong answer raises instead of being timed
    real = h._PIPELINES["fused"]

    def wrong(*a, **k):
        res, spec = real(*a, **k)
        return sw.NonlinearityResult(res.value + 1, res.argmin_v, res.method), spec

    monkeypatch.setitem(h._PIPELINES, "fused", wrong)
    with pytest.raises(sw.BenchVerificationError):
        sw.run_benchmark(sw.generate_sbox(6, 6, 1), ["fused"], repetitions=1)


def test_streamed_spectrum_chunks_match(golden):
    """Chunked, double-buffered export (bounded device memory) equals the
    one-shot spectrum in both layouts, including ragged last chunks."""
    s = box("12x12")
    g = golden["configs"]["12x12"]
    rows, mx = sw.spectrum_to_host(s, chunk_bytes=3 * 4096 * 4 + 7)   # 3 rows per chunk
    assert sha(rows) == g["sha_mask_major"]
    xm, mx2 = sw.spectrum_to_host(s, layout="x", chunk_bytes=1000 * 4096 * 4)
    assert sha(xm) == g["sha_x_major"]
    assert np.array_equal(mx, mx2)
    want, _ = sw.spectrum_device(s, 100, 1100)
    part, _ = sw.spectrum_to_host(s, 100, 1100, chunk_bytes=64 * 4096 * 4)
    assert np.array_equal(part, want.cpu().numpy())


@pytest.mark.slow
def test_16x16_retain_streams_to_host(golden, golden_arrays):
    """fwht_fused(retain) at 16x16: 16 GiB spectrum exported in chunks."""
    s = box("16x16")
    spec, cm = sw.fwht_fused(s, mode="retain")
    assert np.array_equal(cm.values, golden_arrays["maxima_16x16"])
    assert spec.rows.shape == (65535, 65536)
    assert spec.rows[0, :8].tolist() == [0, -368, 440, 104, 52, 348, 260, -196]
    assert spec.rows[-1, :8].tolist() == [0, -296, -56, -104, 272, -128, 288, -40]
    r = sw.nonlinearity_from_spectrum(spec)
    assert (r.value, r.argmin_v) == (31942, 44828)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["20x20", "24x16"])
def test_full_large_config_nl(name):
    """Full 20x20 (2^20 - 1 components) / 24x16 (65535 components) on one GPU,
    EVERY per-component max|W| against a CPU checker:
      * the reference's own full run when it is committed
        (tests/golden/full_<name>.npz, make_golden_full.py: the reference's
        stream body, walsh.py:237-240, over all masks), else
      * the compiled oracle's full arrays (tests/golden/oracle_full_<name>.npz,
        make_oracle_full.py), which tests/test_oracle.py pins to the reference's
        full 16x16 maxima, its sampled masks and every chunk of the reference's
        full run present under tests/golden/full_work/."""
    import json

    gdir = os.path.join(os.path.dirname(__file__), "golden")

    def _has(meta):
        q = os.path.join(gdir, meta)
        return os.path.exists(q) and name in json.load(open(q))["configs"]

    if _has("full_maxima.json"):  # per config: a reference run cut short finalises what it finished
        meta, arr = "full_maxima.json", f"full_{name}.npz"
    elif _has("oracle_full.json"):
        meta, arr = "oracle_full.json", f"oracle_full_{name}.npz"
    else:
        pytest.skip("no full-config goldens (tests/golden/make_oracle_full.py / make_golden_full.py)")
    with open(os.path.join(gdir, meta)) as f:
        g = json.load(f)["configs"][name]
    want = np.load(os.path.join(gdir, arr))["max_abs"]
    s = box(name)
    mx, key = sw.component_max_abs_device(s)
    res = sw.walsh.decode_key(key, s.n)
    assert res == (g["nl"], g["argmin_v"], g["max_abs"])
    full = mx.cpu().numpy()
    assert full.shape == want.shape
    bad = np.flatnonzero(full != want.astype(np.int32))
    assert bad.size == 0, f"{bad.size} components differ, first v = {bad[:5] + 1}"
    _, cm = sw.fwht_fused(s, mode="stream")
    assert sha(cm.values) == g["sha_maxima_i64"]
    # every chunk of the reference's own full run committed so far
    import glob

    for p in glob.glob(os.path.join(gdir, "full_work", f"{name}_*.npy")):
        lo, hi = (int(x) for x in os.path.basename(p)[:-4].split("_")[1:3])
        assert np.array_equal(full[lo - 1:hi - 1], np.load(p).astype(np.int32)), (lo, hi)


def test_evaluate_retain_skips_the_discarded_spectrum():
    """evaluate(method fused/parallel, mode retain) never materialises the
    spectrum it discards, but keeps the reference's retain-mode budget check
    and charge (walsh.py:220-222, parallel.py:91-93) and the same result."""
    s = sw.generate_sbox(12, 12, seed=5, bijective=True)
    need = 4095 * 4096 * 4
    for method in ("fused", "parallel"):
        sw.spectrum_allocations.reset_peak()
        r = sw.evaluate(s, method=method, mode="retain")
        assert sw.spectrum_allocations.peak_bytes >= need and sw.spectrum_allocations.current_bytes == 0
        _, cm = sw.fwht_fused(s, mode="retain")
        assert (r.value, r.argmin_v) == (sw.nonlinearity_from_maxima(cm).value, sw.nonlinearity_from_maxima(cm).argmin_v)
        with pytest.raises(sw.MemoryBudgetError):
            sw.evaluate(s, method=method, mode="retain", max_bytes=need - 1)
    with pytest.raises(ValueError):
        sw.evaluate(s, method="parallel", workers=0)


def test_spectrum_scan_host_chunks_rebase_rows():
    """A host spectrum larger than one scan chunk (256 MiB) is staged chunk by
    chunk; the per-chunk keys are re-based to global rows: largest max|W| wins,
    ties go to the smallest v (nonlinearity.py:36-48)."""
    n = 16
    nrows = 2047  # 2047 x 2^16 int32 = 511.9 MiB: two 256 MiB chunks (1024 + 1023 rows)
    rows = np.zeros((nrows, 1 << n), dtype=np.int32)
    rows[:, 0] = 2
    rows[1000, 5] = -1000   # the maximum, in the first chunk ...
    rows[1100, 7] = 1000    # ... tied by a row of the second chunk
    rows[3, 9] = 998
    r = sw.nonlinearity_from_spectrum(sw.WalshSpectrum(n, 11, rows))
    assert (r.value, r.argmin_v) == (((1 << n) - 1000) // 2, 1001)
    rows[1000, 5] = 0       # now the second chunk holds the unique maximum
    r = sw.nonlinearity_from_spectrum(sw.WalshSpectrum(n, 11, rows))
    assert (r.value, r.argmin_v) == (((1 << n) - 1000) // 2, 1101)
    rows[1000, 5] = -1000
    row_max, _ = sw.nonlinearity.spectrum_row_maxabs(sw.WalshSpectrum(n, 11, rows))
    want = np.abs(rows).max(axis=1)
    assert np.array_equal(row_max.cpu().numpy(), want)


@pytest.mark.parametrize("nrows,chunk_rows", [(7, 3), (64, 64), (65, 8), (1, 5)])
def test_device_to_host_chunked_every_chunk(nrows, chunk_rows):
    """device_to_host_chunked with several chunks and an odd final chunk:
    element-wise equal to a plain device -> host copy."""
    import torch

    src = torch.randint(-2**31, 2**31 - 1, (nrows, 1000), dtype=torch.int32, device="cuda")
    out = np.empty((nrows, 1000), dtype=np.int32)
    sw.walsh.device_to_host_chunked(src, out, chunk_bytes=chunk_rows * 1000 * 4)
    assert np.array_equal(out, src.cpu().numpy())


def test_spectrum_to_host_into_strided_and_read_only_out():
    """spectrum_to_host writes into a caller's negative-stride view with
    numpy's assignment rules and refuses a read-only one like numpy does."""
    s = sw.generate_sbox(9, 6, seed=2)
    want = orc.spectrum(s.table, 9, 1, 64)
    big = np.zeros((63, 512), dtype=np.int32)
    view = big[::-1]
    sw.spectrum_to_host(s, layout="mask", out=view, chunk_bytes=10 * 512 * 4)
    assert np.array_equal(view, want)
    ro = np.zeros((63, 512), dtype=np.int32)
    ro.flags.writeable = False
    with pytest.raises(ValueError):
        sw.spectrum_to_host(s, layout="mask", out=ro)
