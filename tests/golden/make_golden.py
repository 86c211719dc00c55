"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

This script imports the read-only reference package ``sboxeval`` from
``/root/reference/pkg/src`` (it only exists in the build container, never on
the GPU box) and records its outputs.  The committed JSON/NPZ files are what
the tests compare against; nothing at test time reads /root/reference.

Run:  PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--skip-16]

Every number below is produced by calling the reference's own public API:
  generate_sbox            pkg/src/sboxeval/sbox.py:102-111
  fwht_transposed          pkg/src/sboxeval/walsh.py:183-201
  fwht_rowmajor            pkg/src/sboxeval/walsh.py:155-180
  fwht_fused               pkg/src/sboxeval/walsh.py:204-248
  polarity_row             pkg/src/sboxeval/sbox.py:145-152
  fwht_column_in_place     pkg/src/sboxeval/walsh.py:73-104
  nonlinearity_from_*      pkg/src/sboxeval/nonlinearity.py:36-56
  nonlinearity_bruteforce  pkg/src/sboxeval/nonlinearity.py:59-86
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
import sboxeval as se  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


# (name, n, m, bijective) -- BASELINE.json configs, seed 0
CONFIGS = [
    ("8x8", 8, 8, True),
    ("12x12", 12, 12, True),
    ("16x16", 16, 16, True),
    ("20x20", 20, 20, False),
    ("24x16", 24, 16, False),
]


def column_subset(s, masks):
    """Reference stream body (walsh.py:237-240) over a mask subset."""
    pw = 1 << s.n
    buf = np.empty(pw, dtype=np.int32)
    out = []
    for v in masks:
        se.polarity_row(s, v, out=buf)
        w0 = None
        _, max_abs = se.fwht_column_in_place(buf)
        w0 = int(buf[0])
        argmax = int(np.argmax(np.abs(buf.astype(np.int64))))
        out.append({"v": int(v), "max_abs": int(max_abs), "argmax_u": argmax,
                    "w0": w0, "nl": int((pw - max_abs) >> 1),
                    "w_head": [int(x) for x in buf[:8]]})
    return out


def main():
    skip16 = "--skip-16" in sys.argv
    gold = {"generator": "tests/golden/make_golden.py", "numpy": np.__version__,
            "configs": {}, "aes": {}, "small": {}}
    arrays = {}

    # ---- AES (sbox.py:21-38) ---------------------------------------------
    aes = se.aes_sbox()
    spec, cm = se.fwht_fused(aes, mode="retain")
    gold["aes"] = {
        "nl": int(se.nonlinearity_from_maxima(cm).value),
        "argmin_v": int(se.nonlinearity_from_maxima(cm).argmin_v),
        "max_abs": int(np.abs(spec.rows).max()),
        "sha_mask_major": sha(spec.rows),
        "sha_x_major": sha(np.ascontiguousarray(spec.rows.T)),
        "sha_maxima_i64": sha(cm.values),
    }
    arrays["aes_maxima"] = cm.values.astype(np.int64)

    # ---- BASELINE configs, seed 0 -----------------------------------------
    for name, n, m, bij in CONFIGS:
        t0 = time.time()
        s = se.generate_sbox(n, m, seed=0, bijective=bij)
        g = {"n": n, "m": m, "bijective": bij, "seed": 0,
             "table_head": [int(x) for x in s.table[:4]],
             "sha_table_u32": sha(s.table)}
        if n <= 12:
            spec, cm = se.fwht_fused(s, mode="retain")
            nl = se.nonlinearity_from_maxima(cm)
            scan = se.nonlinearity_from_spectrum(spec)
            assert (scan.value, scan.argmin_v) == (nl.value, nl.argmin_v)
            g.update(nl=int(nl.value), argmin_v=int(nl.argmin_v),
                     max_abs=int(np.abs(spec.rows).max()),
                     sha_mask_major=sha(spec.rows),
                     sha_x_major=sha(np.ascontiguousarray(spec.rows.T)),
                     sha_maxima_i64=sha(cm.values),
                     w_v1_head=[int(x) for x in spec.rows[0, :8]],
                     w_vlast_head=[int(x) for x in spec.rows[-1, :8]])
            arrays[f"maxima_{name}"] = cm.values.astype(np.int64)
            if n == 8:
                arrays["spectrum_8x8"] = spec.rows.astype(np.int32)
            rm = se.fwht_rowmajor(s)
            assert np.array_equal(rm.rows, spec.rows)
        elif n == 16 and not skip16:
            _, cm = se.fwht_fused(s, mode="stream")
            nl = se.nonlinearity_from_maxima(cm)
            g.update(nl=int(nl.value), argmin_v=int(nl.argmin_v),
                     max_abs=int((1 << n) - 2 * int(nl.value)),
                     sha_maxima_i64=sha(cm.values))
            arrays["maxima_16x16"] = cm.values.astype(np.int64)
        if n >= 16:
            sub = list(range(1, 9)) + [(1 << m) - 1]
            g["subset"] = column_subset(s, sub)
        g["ref_seconds"] = round(time.time() - t0, 2)
        gold["configs"][name] = g
        print(name, g.get("nl"), g["ref_seconds"], "s", flush=True)

    # ---- small-box sweep (test_acceptance.py:61-90 shapes, seeds 0..49) ----
    sweep = []
    for n, m in [(3, 3), (4, 4), (5, 5), (6, 4), (4, 6), (1, 1), (1, 3), (2, 5),
                 (3, 8), (5, 9), (4, 7), (7, 3), (9, 5), (10, 10), (11, 6), (13, 3),
                 (14, 2), (15, 2), (16, 1), (6, 11)]:
        seeds = range(50) if n <= 6 and m <= 6 else range(3)
        for seed in seeds:
            for bij in ((False, True) if n == m and seed < 2 else (False,)):
                s = se.generate_sbox(n, m, seed, bijective=bij)
                spec, cm = se.fwht_fused(s, mode="retain")
                nl = se.nonlinearity_from_maxima(cm)
                rec = {"n": n, "m": m, "seed": seed, "bijective": bij,
                       "sha_table_u32": sha(s.table),
                       "nl": int(nl.value), "argmin_v": int(nl.argmin_v),
                       "sha_mask_major": sha(spec.rows),
                       "sha_maxima_i64": sha(cm.values)}
                if n <= 8 and m <= 8:
                    rec["nl_bruteforce"] = int(se.nonlinearity_bruteforce(s).value)
                sweep.append(rec)
    gold["small"]["sweep"] = sweep

    # identity / constant / affine boxes (sbox.py:98-99; test_nonlinearity.py:70-78)
    specials = []
    for label, s in [("identity4", se.identity_sbox(4)),
                     ("identity10", se.identity_sbox(10)),
                     ("constant5x3", se.SBox(5, 3, np.zeros(32, dtype=np.uint32))),
                     ("affine4", se.SBox(4, 4, np.arange(16, dtype=np.uint32) ^ 0b1011))]:
        spec, cm = se.fwht_fused(s, mode="retain")
        nl = se.nonlinearity_from_maxima(cm)
        specials.append({"label": label, "n": s.n, "m": s.m,
                         "table": [int(x) for x in s.table] if s.n <= 5 else None,
                         "nl": int(nl.value), "argmin_v": int(nl.argmin_v),
                         "sha_mask_major": sha(spec.rows),
                         "sha_maxima_i64": sha(cm.values)})
    gold["small"]["specials"] = specials

    # ---- fwht_column_in_place on general int32 columns (walsh.py:73-104) ----
    cols = []
    for k in range(0, 15):
        rng = np.random.default_rng(1000 + k)
        vals = rng.integers(-5, 6, size=1 << k).astype(np.int32)
        col = vals.copy()
        _, mx = se.fwht_column_in_place(col)
        arrays[f"col_in_{k}"] = vals
        cols.append({"k": k, "max_abs": int(mx), "sha_out": sha(col)})
    # wide-range column: int32 wraparound semantics of numpy
    rng = np.random.default_rng(7)
    big = rng.integers(-(1 << 30), 1 << 30, size=1 << 10).astype(np.int32)
    col = big.copy()
    _, mx = se.fwht_column_in_place(col)
    arrays["col_in_wrap"] = big
    cols.append({"k": 10, "label": "wrap", "max_abs": int(mx), "sha_out": sha(col)})
    gold["small"]["columns"] = cols

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(gold, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "golden_arrays.npz"), **arrays)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
