"""One-off stress of the n = 16 NL kernels against the compiled CPU oracle:
random boxes (random and structured), widths m = 1..24 and mask ranges incl. ranges that
start / end inside Gray blocks, 1-3 mask ranges and > 148 * k masks.  Not part of the test
suite (tests/test_gpu_tc16.py::test_random_ranges_n16 runs 12 such trials).
    python tools/lut_stress.py [trials]"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw  # noqa: E402
from oracle import sbw_oracle as orc  # noqa: E402

trials = int(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(20261021)
bad = 0
for t in range(trials):
    m = int(rng.integers(1, 25))
    kind = int(rng.integers(0, 5))
    x = np.arange(1 << 16, dtype=np.uint32)
    if kind == 0:      # affine-heavy: low bits of S are linear in x
        tab = (x ^ (x >> 3) ^ int(rng.integers(0, 1 << 16))) & ((1 << m) - 1)
        tab = tab.astype(np.uint32)
        s = sw.SBox(16, m, tab)
    elif kind == 1:    # constant / near-constant components
        tab = np.where(rng.random(1 << 16) < 0.001, rng.integers(0, 1 << m, 1 << 16), 0).astype(np.uint32)
        s = sw.SBox(16, m, tab)
    else:
        s = sw.generate_sbox(16, m, int(rng.integers(0, 1 << 30)), bijective=(m == 16))
    top = 1 << m
    lo = int(rng.integers(1, top))
    span = int(rng.choice([1, 2, 3, 147, 148, 149, 255, 256, 257, 300, 1000, 3000]))
    hi = int(min(top, lo + span))
    mx, key = sw.component_max_abs_device(s, lo, hi)
    got = mx.cpu().numpy()
    want = orc.component_max_abs_c(np.asarray(s.table), 16, lo, hi) if hasattr(orc, "component_max_abs_c") else orc.component_max_abs(s.table, 16, lo, hi)
    res = sw.walsh.decode_key(key, 16)
    i = int(np.argmax(want))
    ok = np.array_equal(got, want) and (res[1], res[2]) == (lo + i, int(want[i]))
    if not ok:
        bad += 1
        print("MISMATCH", t, m, kind, lo, hi, np.flatnonzero(got != want)[:5], flush=True)
print(f"{trials} trials, {bad} mismatches")
