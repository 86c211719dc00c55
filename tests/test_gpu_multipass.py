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
    assert sw.walsh.decode_key(key, n)[:2] == (0, 1)  # NL 0, first v wins ties


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


# ---- the L2 ring (SBW_K3_RING=1): concurrent pass A / pass B ---------------
# Off by default (measured slower, K3); kept exact.  The ring
# reorders components (Gray order per pass-A CTA row, slot positions per
# batch) and hands batches between two co-resident kernels, so every case
# compares the whole maxima array and the key with the batched path and
# samples masks against the oracle; ranges leave a tail for the batched path.
@pytest.mark.parametrize("n,m,bij,lo,hi,na,L,R", [
    (20, 20, False, 1, 3001, 64, 4, 3),      # 187 batches of 16 + a tail of 8
    (17, 17, True, 5, 4100, 64, 2, 3),       # T = 2: 32 CTAs per block pair
    (21, 12, False, 1, 4096, 64, 1, 2),      # T = 32: 2 CTAs per block pair, L = 1
    (19, 16, False, 300, 9000, 96, 3, 4),    # L not a power of two, unaligned start
])
def test_ring_matches_batched(monkeypatch, n, m, bij, lo, hi, na, L, R):
    s = sw.generate_sbox(n, m, seed=n + m, bijective=bij)
    monkeypatch.setenv("SBW_K3_RING", "0")
    want_mx, want_key = sw.component_max_abs_device(s, lo, hi)
    monkeypatch.setenv("SBW_K3_RING", "1")
    monkeypatch.setenv("SBW_K3_NA", str(na))
    monkeypatch.setenv("SBW_K3_RING_L", str(L))
    monkeypatch.setenv("SBW_K3_RING_R", str(R))
    got_mx, got_key = sw.component_max_abs_device(s, lo, hi)
    got = got_mx.cpu().numpy()
    assert np.array_equal(got, want_mx.cpu().numpy())
    assert int(got_key.item()) == int(want_key.item())
    rng = np.random.default_rng(n)
    for v in sorted(set(rng.integers(lo, hi, size=3).tolist()) | {lo, hi - 1}):
        assert int(got[v - lo]) == int(orc.component_max_abs(s.table, n, v, v + 1)[0]), v


# ---- 16 stages in pass A (SBW_K3_EMIT16=1, off by default) --------------------
# Pass A also runs stage 16 and writes the wrapped u16; a batch in which a tile
# wrapped (|W_16| = 2^16: affine on the tile) is redone by gated 15-stage
# launches.  Linear components wrap in every tile (all fallback); random ones
# never do (all 16-stage); both must match the default path and the oracle.
@pytest.mark.parametrize("n,m,seed,lo,hi", [(18, 18, 21, 1, 3000), (20, 12, 22, 1, 4096),
                                             (21, 16, 23, 100, 400), (24, 16, 24, 1, 9)])
def test_emit16_random_matches_default(monkeypatch, n, m, seed, lo, hi):
    s = sw.generate_sbox(n, m, seed, bijective=False)
    monkeypatch.setenv("SBW_K3_EMIT16", "0")
    want, wkey = sw.component_max_abs_device(s, lo, hi)
    monkeypatch.setenv("SBW_K3_EMIT16", "1")
    got, gkey = sw.component_max_abs_device(s, lo, hi)
    assert np.array_equal(got.cpu().numpy(), want.cpu().numpy()) and int(gkey.item()) == int(wkey.item())
    v = lo + (hi - lo) // 2
    assert int(got[v - lo].item()) == int(orc.component_max_abs(s.table, n, v, v + 1)[0])


@pytest.mark.parametrize("n", [18, 20, 21, 24])
def test_emit16_linear_components_fall_back(monkeypatch, n):
    monkeypatch.setenv("SBW_K3_EMIT16", "1")
    s = _linear_sbox(n)
    mx, key = sw.component_max_abs_device(s)
    assert np.all(mx.cpu().numpy() == 1 << n)
    assert sw.walsh.decode_key(key, n)[:2] == (0, 1)


_LUT_EMIT_ARM = r"""
import json, sys, hashlib
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1912_03732_b200 as sw
out = {}
for n, m, lo, hi in [(17, 8, 1, 256), (18, 18, 1000, 3000), (20, 20, 1, 5000), (21, 16, 7, 300), (24, 16, 1, 40)]:
    s = sw.generate_sbox(n, m, n + m, bijective=False)
    mx, key = sw.component_max_abs_device(s, lo, hi)
    out[f"{n},{m}"] = [hashlib.sha256(mx.cpu().numpy().tobytes()).hexdigest(), int(key.item())]
lin = sw.SBox(17, 8, np.arange(1 << 17, dtype=np.uint32) & 0xFF)   # linear components: W = +2^17 at one u
mx, key = sw.component_max_abs_device(lin, 1, 256)
out["linear17"] = [int(mx.min()), int(mx.max())]
print(json.dumps(out))
"""


def test_table_lookup_pass_a_matches_default():
    """k_tc_lut_emit (SBW_TC_LUT_EMIT=1, off by default: exact but slower) writes the
    same pass-A scratch contents up to its block-internal order: maxima and keys
    equal those of the default k_tc_hybrid<EMIT> path, incl. the |W| = 2^n extreme."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for arm in ("1", "0"):
        p = subprocess.run(["timeout", "300", sys.executable, "-c", _LUT_EMIT_ARM, root],
                           env=dict(os.environ, SBW_TC_LUT_EMIT=arm), capture_output=True, text=True)
        assert p.returncode == 0, p.stderr[-2000:]
        res[arm] = json.loads(p.stdout.strip().splitlines()[-1])
    assert res["1"] == res["0"]
    assert res["1"]["linear17"] == [1 << 17, 1 << 17]
