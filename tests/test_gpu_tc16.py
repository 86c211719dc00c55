"""Parity of the n = 16 tensor-core kernel (k_tc_hybrid<NL>, sbw_tc.cu).

sbw_nl at n = 16 runs the hybrid kernel: x bits 0..7 and the c0 butterfly as
an int8 tcgen05 GEMM, x bits 9..15 as packed integer stages.  These cases target what is specific to
it -- the u = 0 row correction, the Gray-code mask order inside aligned
blocks of 256, CTA ranges of one or two masks, m > 16 -- and cross-check it
against the all-ALU tile kernel (SBW_TC=0, k_tile_simd) on the same inputs.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1912_03732_b200 as sw
from oracle import sbw_oracle as orc

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _maxima(s, lo, hi):
    mx, key = sw.component_max_abs_device(s, lo, hi)
    return mx.cpu().numpy().astype(np.int64), sw.walsh.decode_key(key, s.n)


def test_constant_components_w0_extremes():
    """Bit 15 of S is constant 1 and bit 14 constant 0: the components v =
    0x8000 and 0x4000 are constant, so the maximum is W(0) = -2^16 / +2^16 --
    the coefficient that carries the row u = 0 correction."""
    rng = np.random.default_rng(5)
    t = (rng.integers(0, 1 << 14, 1 << 16, dtype=np.uint32) | 0x8000)
    s = sw.SBox(16, 16, t)
    for lo, hi in [(0x4000 - 3, 0x4000 + 3), (0x8000 - 2, 0x8000 + 5), (0xC000 - 1, 0xC000 + 1)]:
        got, _ = _maxima(s, lo, hi)
        assert np.array_equal(got, orc.component_max_abs(s.table, 16, lo, hi))
    got, _ = _maxima(s, 0x8000, 0x8001)
    assert got[0] == 1 << 16


@pytest.mark.parametrize("lo,hi", [(1, 2), (1, 149), (1, 297), (255, 258), (256, 512),
                                   (200, 1000), (65280, 65536), (12345, 12345 + 777)])
def test_ranges_and_gray_blocks(lo, hi):
    """One or two masks per CTA, ranges that start/end inside aligned blocks
    of 256 (natural order there) and whole blocks (Gray-code order)."""
    s = sw.generate_sbox(16, 16, 21, bijective=True)
    got, (nl, v, m) = _maxima(s, lo, hi)
    want = orc.component_max_abs(s.table, 16, lo, hi)
    assert np.array_equal(got, want)
    i = int(np.argmax(want))  # first maximum = smallest v
    assert (v, m) == (lo + i, int(want[i]))
    assert nl == ((1 << 16) - int(want[i])) // 2


@pytest.mark.parametrize("m", [1, 5, 20, 24])
def test_output_widths(m):
    s = sw.generate_sbox(16, m, 3 + m, bijective=False)
    hi = min(1 << m, 700)
    got, _ = _maxima(s, 1, hi)
    assert np.array_equal(got, orc.component_max_abs(s.table, 16, 1, hi))


_ARM = r'''
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1912_03732_b200 as sw
out = {}
for seed, m, lo, hi in [(0, 16, 1, 65536), (9, 18, 1, 40000), (4, 16, 999, 4242)]:
    s = sw.generate_sbox(16, m, seed, bijective=(m == 16))
    mx, key = sw.component_max_abs_device(s, lo, hi)
    out[f"{seed},{m},{lo},{hi}"] = [mx.cpu().numpy().astype(np.int64).tolist(), int(key.item())]
print(json.dumps(out))
'''


def test_tensor_core_kernel_matches_alu_kernel():
    """Same maxima and key from the four n = 16 NL kernels: k_tc_lut16 (default),
    its 8-warp form k_tc_lut (SBW_LUT_WARPS=8), k_tc_hybrid<NL> (SBW_TC_LUT=0) and
    the all-ALU k_tile_simd<16> (SBW_TC=0)."""
    res = {}
    for arm, env in (("lut", {}), ("lut8", {"SBW_LUT_WARPS": "8"}), ("hybrid", {"SBW_TC_LUT": "0"}),
                     ("alu", {"SBW_TC": "0"})):
        p = subprocess.run([sys.executable, "-c", _ARM, ROOT], env=dict(os.environ, **env),
                           capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        res[arm] = json.loads(p.stdout.strip().splitlines()[-1])
    assert res["lut"] == res["alu"]
    assert res["lut8"] == res["alu"]
    assert res["hybrid"] == res["alu"]


def test_live_peak_microbenchmarks():
    """The roofline denominators bench.py measures live: int32 lane-ops and
    tcgen05 kind::i8 MMA throughput, both in a sane range for a B200."""
    import ctypes

    import paper_1912_03732_b200.device as d

    lib = d.load_library()
    for fn, lo, hi in (("sbw_int32_peak", 5e12, 2e14), ("sbw_int8_mma_peak", 1e15, 1e16)):
        ops, ms = ctypes.c_double(0), ctypes.c_double(0)
        d.check(getattr(lib, fn)(ctypes.byref(ops), ctypes.byref(ms), None))
        assert lo < ops.value < hi, (fn, ops.value)
        assert ms.value > 0


@pytest.mark.parametrize("trial", range(12))
def test_random_ranges_n16(trial):
    """Random S-boxes, widths and mask ranges through the tensor-core kernel."""
    rng = np.random.default_rng(1000 + trial)
    m = int(rng.integers(1, 25))
    s = sw.generate_sbox(16, m, int(rng.integers(0, 1 << 30)), bijective=(m == 16))
    top = 1 << m
    lo = int(rng.integers(1, top))
    hi = int(min(top, lo + rng.integers(1, 600)))
    got, (nl, v, mxw) = _maxima(s, lo, hi)
    want = orc.component_max_abs(s.table, 16, lo, hi)
    assert np.array_equal(got, want)
    i = int(np.argmax(want))
    assert (v, mxw) == (lo + i, int(want[i]))


@pytest.mark.parametrize("n,m,seed,lo,hi", [(17, 9, 1, 1, 40), (18, 12, 2, 100, 140), (19, 5, 3, 1, 32),
                                             (20, 20, 4, 777, 800), (21, 16, 5, 1, 12), (24, 16, 6, 60000, 60004)])
def test_multipass_tensor_core_pass_a(n, m, seed, lo, hi):
    """n = 17..24 NL: the tensor-core pass A (k_tc_hybrid<EMIT>) + pass B."""
    s = sw.generate_sbox(n, m, seed, bijective=False)
    got, _ = _maxima(s, lo, hi)
    assert np.array_equal(got, orc.component_max_abs(s.table, n, lo, hi))


@pytest.mark.parametrize("n,m,lo,hi", [(15, 1, 1, 2), (15, 15, 1, 1 << 15), (14, 2, 1, 4), (14, 14, 5, 3001),
                                       (13, 3, 1, 8), (13, 16, 1000, 1901), (12, 4, 1, 16), (12, 12, 1, 4096),
                                       (11, 5, 1, 32), (11, 11, 17, 2000), (11, 20, 123456, 124000)])
def test_small_n_tensor_core_slots(n, m, lo, hi):
    """n = 12..15 NL packs 2^(16-n) components per tile (slots); ranges that
    start / end inside an item, the item holding v = 0, m = 16 - n exactly.
    (n = 11 runs on the tile kernel in the default 16-row-generation build and
    on the tensor cores in an SBW_TC_ROWS=8 build; same expectations.)"""
    s = sw.generate_sbox(n, m, 40 + n, bijective=(n == m))
    got, (nl, v, mxw) = _maxima(s, lo, hi)
    want = orc.component_max_abs(s.table, n, lo, hi)
    assert np.array_equal(got, want)
    i = int(np.argmax(want))
    assert (v, mxw) == (lo + i, int(want[i]))


@pytest.mark.parametrize("n,m,lo,hi", [(15, 15, 1, 700), (14, 14, 5, 1001), (13, 16, 1000, 1301),
                                       (12, 12, 1, 4096), (12, 4, 1, 16), (15, 1, 1, 2), (14, 20, 70001, 70040)])
def test_small_n_tensor_core_spectrum(n, m, lo, hi):
    """n = 12..15 materialised spectra on the tensor-core kernel (k_tc_hybrid<SPEC, n>):
    exact W per slot, ranges starting / ending inside an item, m = 16 - n exactly."""
    s = sw.generate_sbox(n, m, 60 + n, bijective=(n == m))
    rows, mx = sw.spectrum_device(s, lo, hi)
    want = orc.spectrum(s.table, n, lo, hi)
    assert np.array_equal(rows.cpu().numpy(), want)
    assert np.array_equal(mx.cpu().numpy(), np.abs(want).max(axis=1))
