"""Multi-pass path (n = 17..24, K3): pass A + the fp32 pass B kernels.

Pass B runs its butterflies in fp32 (sbw_passb.cuh, lo_half_f): exact only
because every intermediate stays an integer of magnitude <= 2^23.  These
cases drive it to that bound -- constant and linear components, whose only
nonzero coefficient is W = +2^n -- at every H = n - 15 (both k_passb_regs,
H <= 5, and every k_passb_staged shape, H = 6..9), in the max path and in
the retained spectrum, and cross-check random S-boxes at the H values the
other suites do not cover.
"""
import numpy as np
import pytest

import paper_1912_03732_b200 as sw
from oracle import sbw_oracle as orc

pytestmark = pytest.mark.gpu


def _linear_sbox(n):
    """S(x) = x_{n-1} | x_0 << 1 | 0 << 2: components v = 1..7 are g_v(x) =
    <a_v, x> with a_v in {0, 1, 2^(n-1), 2^(n-1) + 1}; W(u, v) = 2^n at u = a_v
    and 0 elsewhere (walsh.py:56-70)."""
    x = np.arange(1 << n, dtype=np.uint32)
    return sw.SBox(n, 3, ((x >> (n - 1)) & 1) | ((x & 1) << 1))


def _a_of(v, n):
    return (((v >> 0) & 1) << (n - 1)) | ((v >> 1) & 1)


@pytest.mark.parametrize("n", list(range(17, 25)))
def test_linear_components_reach_2_pow_n(n):
    s = _linear_sbox(n)
    mx, key = sw.component_max_abs_device(s)
    assert np.all(mx.cpu().numpy() == 1 << n)
    assert sw.transforms.decode_key(key, n)[:2] == (0, 1)  # NL 0, first v wins ties


@pytest.mark.parametrize("n", [17, 20, 21, 23])
def test_retained_spectrum_single_spike(n):
    s = _linear_sbox(n)
    spec, cm = sw.fwht_fused(s, mode="retain")
    rows = np.asarray(spec.rows)
    assert rows.shape == (7, 1 << n)
    for v in range(1, 8):
        row = rows[v - 1]
        nz = np.flatnonzero(row)
        assert nz.tolist() == [_a_of(v, n)], (v, nz[:4])
        assert int(row[nz[0]]) == 1 << n
    assert np.all(np.asarray(cm.values) == 0)  # per-component NL = 2^(n-1) - max/2


@pytest.mark.parametrize("n,m,seed,lo,hi", [(22, 10, 11, 1, 4), (23, 8, 12, 200, 203),
                                             (20, 4, 13, 1, 16), (22, 22, 14, 4194300, 4194304)])
def test_random_against_oracle(n, m, seed, lo, hi):
    s = sw.generate_sbox(n, m, seed, bijective=False)
    mx, _ = sw.component_max_abs_device(s, lo, hi)
    assert np.array_equal(mx.cpu().numpy().astype(np.int64), orc.component_max_abs(s.table, n, lo, hi))
