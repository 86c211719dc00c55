"""Pin the CPU oracle (oracle/sbw_oracle.py) to the reference's own outputs.

tests/golden/* were produced by tests/golden/make_golden.py running the
reference package itself; every oracle function the GPU tests rely on is
checked here against them.  CPU only.
"""
import numpy as np
import pytest

from oracle import sbw_oracle as orc
from tests.util import sha

CFG = {"8x8": (8, 8, True), "12x12": (12, 12, True), "16x16": (16, 16, True),
       "20x20": (20, 20, False), "24x16": (24, 16, False)}


@pytest.mark.parametrize("name", list(CFG))
def test_seeded_tables_match_reference(golden, name):
    n, m, bij = CFG[name]
    t = orc.gen_table(n, m, 0, bij)
    g = golden["configs"][name]
    assert sha(t) == g["sha_table_u32"]
    assert t[:4].tolist() == g["table_head"]


def test_aes_spectrum_and_maxima(golden):
    from paper_1912_03732_b200 import AES_SBOX

    t = np.array(AES_SBOX, dtype=np.uint32)
    rows = orc.spectrum(t, 8, 1, 256)
    g = golden["aes"]
    assert sha(rows) == g["sha_mask_major"]
    assert sha(np.ascontiguousarray(rows.T)) == g["sha_x_major"]
    nl = orc.component_nl(t, 8, 1, 256)
    assert sha(nl) == g["sha_maxima_i64"]
    assert orc.nl_from_maxima(nl) == (g["nl"], g["argmin_v"]) == (112, 1)
    assert orc.nl_from_spectrum(rows, 8) == (112, 1)
    assert int(np.abs(rows).max()) == 32


@pytest.mark.parametrize("name", ["8x8", "12x12"])
def test_materialised_configs(golden, golden_arrays, name):
    n, m, bij = CFG[name]
    t = orc.gen_table(n, m, 0, bij)
    g = golden["configs"][name]
    rows = orc.spectrum(t, n, 1, 1 << m)
    assert sha(rows) == g["sha_mask_major"]
    assert sha(np.ascontiguousarray(rows.T)) == g["sha_x_major"]
    assert rows[0, :8].tolist() == g["w_v1_head"]
    assert rows[-1, :8].tolist() == g["w_vlast_head"]
    nl = orc.component_nl(t, n, 1, 1 << m)
    assert sha(nl) == g["sha_maxima_i64"]
    assert np.array_equal(nl, golden_arrays[f"maxima_{name}"])
    assert orc.nl_from_maxima(nl) == (g["nl"], g["argmin_v"])
    assert orc.nl_from_spectrum(rows, n) == (g["nl"], g["argmin_v"])


def test_16x16_maxima_subset(golden, golden_arrays):
    t = orc.gen_table(16, 16, 0, True)
    full = golden_arrays["maxima_16x16"]
    assert sha(full) == golden["configs"]["16x16"]["sha_maxima_i64"]
    assert orc.nl_from_maxima(full) == (31942, 44828)
    assert np.array_equal(orc.component_nl(t, 16, 1, 65), full[:64])
    assert np.array_equal(orc.component_nl(t, 16, 44828, 44829), full[44827:44828])
    assert np.array_equal(orc.component_nl(t, 16, 65535, 65536), full[-1:])


@pytest.mark.parametrize("name,masks", [("20x20", 8), ("24x16", 2)])
def test_large_config_subsets(golden, name, masks):
    n, m, bij = CFG[name]
    t = orc.gen_table(n, m, 0, bij)
    sub = [r for r in golden["configs"][name]["subset"] if r["v"] <= masks]
    for rec in sub:
        v = rec["v"]
        row = orc.spectrum(t, n, v, v + 1)[0]
        assert int(np.abs(row).max()) == rec["max_abs"]
        assert int(np.argmax(np.abs(row.astype(np.int64)))) == rec["argmax_u"]
        assert row[:8].tolist() == rec["w_head"]
        assert orc.column_nl(1 << n, rec["max_abs"]) == rec["nl"]


def test_small_sweep(golden):
    for rec in golden["small"]["sweep"]:
        n, m = rec["n"], rec["m"]
        t = orc.gen_table(n, m, rec["seed"], rec["bijective"])
        assert sha(t) == rec["sha_table_u32"]
        rows = orc.spectrum(t, n, 1, 1 << m)
        assert sha(rows) == rec["sha_mask_major"], rec
        nl = orc.component_nl(t, n, 1, 1 << m)
        assert sha(nl) == rec["sha_maxima_i64"]
        assert orc.nl_from_maxima(nl) == (rec["nl"], rec["argmin_v"])
        if "nl_bruteforce" in rec and n <= 6 and m <= 6:
            assert orc.nl_bruteforce(t, n, m)[0] == rec["nl_bruteforce"]


def test_specials(golden):
    from paper_1912_03732_b200 import identity_sbox

    for rec in golden["small"]["specials"]:
        if rec["table"] is not None:
            t = np.array(rec["table"], dtype=np.uint32)
        else:
            t = identity_sbox(rec["n"]).table
        rows = orc.spectrum(t, rec["n"], 1, 1 << rec["m"])
        assert sha(rows) == rec["sha_mask_major"], rec["label"]
        nl = orc.component_nl(t, rec["n"], 1, 1 << rec["m"])
        assert orc.nl_from_maxima(nl) == (rec["nl"], rec["argmin_v"])


def test_general_columns(golden, golden_arrays):
    for rec in golden["small"]["columns"]:
        key = "col_in_wrap" if rec.get("label") == "wrap" else f"col_in_{rec['k']}"
        out, mx = orc.fwht_column(golden_arrays[key])
        assert sha(out) == rec["sha_out"], rec
        assert mx == rec["max_abs"], rec


def test_known_answer_columns():
    out, mx = orc.fwht_column(np.array([1, 1, 1, -1], dtype=np.int32))
    assert out.tolist() == [2, 2, 2, -2] and mx == 2
    out, mx = orc.fwht_column(np.array([-7], dtype=np.int32))
    assert out.tolist() == [-7] and mx == 7
    with pytest.raises(ValueError, match="power of two"):
        orc.fwht_column(np.ones(6, dtype=np.int32))


def test_walsh_direct_matches_spectrum():
    t = orc.gen_table(5, 4, 9)
    rows = orc.spectrum(t, 5, 1, 16)
    for v in range(1, 16):
        for u in range(32):
            assert orc.walsh_direct(t, 5, u, v) == rows[v - 1, u]


def test_stream_loop_equals_batched():
    t = orc.gen_table(9, 7, 3)
    assert np.array_equal(orc.stream_loop(t, 9, 1, 128), orc.component_nl(t, 9, 1, 128))


def test_partition():
    assert [b - a for a, b in orc.partition_columns(15, 8)] == [2, 2, 2, 2, 2, 2, 2, 1]
    assert orc.partition_columns(3, 8) == ((1, 2), (2, 3), (3, 4))


# ---- column API on every integer dtype / x-major (golden_api.*, produced by
# ---- tests/golden/make_golden_api.py running the reference) ---------------
def _api():
    import json
    import os

    here = os.path.join(os.path.dirname(__file__), "golden")
    with open(os.path.join(here, "golden_api.json")) as f:
        meta = json.load(f)
    with np.load(os.path.join(here, "golden_api.npz")) as z:
        arrays = {k: z[k] for k in z.files}
    return meta, arrays


def test_typed_columns_oracle_matches_reference():
    meta, arrays = _api()
    for rec in meta["columns"]:
        col = arrays[rec["key"] + "_in"]
        out, mx = orc.fwht_column_typed(col)
        assert out.dtype == col.dtype
        assert np.array_equal(out, arrays[rec["key"] + "_out"]), rec
        assert mx == rec["max_abs"], rec


def test_xmajor_oracle_matches_reference():
    meta, _ = _api()
    for rec in meta["xmajor"]:
        t = orc.gen_table(rec["n"], rec["m"], rec["seed"], rec["bijective"])
        wt = np.ascontiguousarray(orc.polarity_block(t, 1, 1 << rec["m"]).T)
        assert sha(wt) == rec["sha_polarity_xmajor"]
        assert sha(orc.xmajor_spectrum_typed(wt)) == rec["sha_spectrum_xmajor"]
    for pw, mx, nl in meta["column_nonlinearity"]:
        assert orc.column_nl(pw, mx) == nl


@pytest.mark.parametrize("name,masks", [("20x20", (1, 2, 3, 334146, 1048575)), ("24x16", (1, 27804, 65535))])
def test_full_large_config_goldens(name, masks):
    """The oracle against the reference's full per-component maxima of the two
    large configs (tests/golden/full_<name>.npz, make_golden_full.py): the
    overall NL / argmin and a few components including the argmin."""
    import json
    import os

    here = os.path.join(os.path.dirname(__file__), "golden")
    if not os.path.exists(os.path.join(here, "full_maxima.json")):
        pytest.skip("tests/golden/full_maxima.json not generated yet (tests/golden/make_golden_full.py)")
    cfgs = json.load(open(os.path.join(here, "full_maxima.json")))["configs"]
    if name not in cfgs:
        pytest.skip(f"the reference's full {name} run is not complete yet (chunks under tests/golden/full_work/)")
    g = cfgs[name]
    full = np.load(os.path.join(here, f"full_{name}.npz"))["max_abs"].astype(np.int64)
    n, m, bij = CFG[name]
    assert full.shape == ((1 << m) - 1,)
    values = ((1 << n) - full) >> 1
    assert sha(values) == g["sha_maxima_i64"]
    assert orc.nl_from_maxima(values) == (g["nl"], g["argmin_v"])
    t = orc.gen_table(n, m, 0, bij)
    for v in masks:
        assert int(orc.component_max_abs(t, n, v, v + 1)[0]) == int(full[v - 1]), v


# ---- the compiled oracle (oracle/sbw_oracle.c) ------------------------------
def _c_oracle_or_skip():
    import os

    if not os.path.exists(os.path.join(os.path.dirname(orc.__file__), "liboracle.so")):
        pytest.skip("oracle/liboracle.so not built (make -C oracle)")


def test_c_oracle_full_16x16_matches_reference(golden, golden_arrays):
    """Every one of the 65535 16x16 maxima, C oracle vs the reference's run."""
    _c_oracle_or_skip()
    t = orc.gen_table(16, 16, 0, True)
    mx = orc.component_max_abs_c(t, 16, 1, 1 << 16)
    assert np.array_equal(((1 << 16) - mx) >> 1, golden_arrays["maxima_16x16"])


@pytest.mark.parametrize("n,m,bij,seed", [(1, 1, False, 0), (2, 3, False, 1), (5, 4, False, 9),
                                           (8, 8, True, 0), (11, 3, False, 2), (13, 6, False, 4),
                                           (14, 2, False, 5)])
def test_c_oracle_small_shapes(n, m, bij, seed):
    _c_oracle_or_skip()
    t = orc.gen_table(n, m, seed, bij)
    for threads in (1, 3):
        assert np.array_equal(orc.component_max_abs_c(t, n, 1, 1 << m, threads),
                              orc.component_max_abs(t, n, 1, 1 << m))
    assert orc.component_max_abs_c(t, n, 1, 1).shape == (0,)


def test_c_oracle_large_subsets_match_reference(golden):
    """The reference's sampled 20x20 / 24x16 masks (make_golden.py)."""
    _c_oracle_or_skip()
    for name in ("20x20", "24x16"):
        n, m, bij = CFG[name]
        t = orc.gen_table(n, m, 0, bij)
        for rec in golden["configs"][name]["subset"]:
            v = rec["v"]
            assert int(orc.component_max_abs_c(t, n, v, v + 1)[0]) == rec["max_abs"], (name, v)


def _reference_chunks(name):
    """Chunks of the reference's own full run (make_golden_full.py) present."""
    import glob
    import os

    here = os.path.join(os.path.dirname(__file__), "golden", "full_work")
    out = []
    for p in sorted(glob.glob(os.path.join(here, f"{name}_*.npy"))):
        lo, hi = (int(x) for x in os.path.basename(p)[:-4].split("_")[1:3])
        out.append((lo, hi, np.load(p)))
    return out


@pytest.mark.parametrize("name", ["20x20", "24x16"])
def test_oracle_full_arrays_match_every_reference_chunk(name):
    """tests/golden/oracle_full_<name>.npz (every component, from the C oracle)
    equals the reference's own maxima on every chunk its full run has produced,
    and the final full_<name>.npz when that run has finished."""
    import json
    import os

    here = os.path.join(os.path.dirname(__file__), "golden")
    path = os.path.join(here, f"oracle_full_{name}.npz")
    if not os.path.exists(path):
        pytest.skip("tests/golden/oracle_full_*.npz not generated (make_oracle_full.py)")
    n, m, _ = CFG[name]
    full = np.load(path)["max_abs"].astype(np.int64)
    assert full.shape == ((1 << m) - 1,)
    meta = json.load(open(os.path.join(here, "oracle_full.json")))["configs"][name]
    values = ((1 << n) - full) >> 1
    assert sha(values) == meta["sha_maxima_i64"]
    assert orc.nl_from_maxima(values) == (meta["nl"], meta["argmin_v"])
    covered = 0
    for lo, hi, chunk in _reference_chunks(name):
        assert np.array_equal(chunk.astype(np.int64), full[lo - 1:hi - 1]), (name, lo, hi)
        covered += hi - lo
    ref_full = os.path.join(here, f"full_{name}.npz")
    if os.path.exists(ref_full):
        assert np.array_equal(np.load(ref_full)["max_abs"].astype(np.int64), full)
        covered = full.shape[0]
    print(f"{name}: reference covers {covered} of {full.shape[0]} components")
