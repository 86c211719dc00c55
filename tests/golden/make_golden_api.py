"""Golden fixtures for the column/x-major API surface, produced by the REFERENCE.

Covers the reference functions whose round-1 GPU counterparts were missing
or int32-only:
  fwht_column_in_place   pkg/src/sboxeval/walsh.py:73-104  (every integer dtype,
                         strided views, wrap-around, length 1)
  column_nonlinearity    pkg/src/sboxeval/walsh.py:107-114
  build_polarity_xmajor  pkg/src/sboxeval/walsh.py:117-131
  transform_xmajor_in_place  pkg/src/sboxeval/walsh.py:134-137
  transform_rows_in_place    pkg/src/sboxeval/walsh.py:140-152 (maxima_out)

Writes tests/golden/golden_api.npz (inputs + reference outputs) and
golden_api.json (max_abs values, shas).  Build container only (imports
/root/reference); run:  PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_api.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import sboxeval as se  # noqa: E402
import sboxeval.walsh as sw_ref  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
DTYPES = ["int8", "uint8", "int16", "uint16", "int32", "uint32", "int64", "uint64"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def main():
    rng = np.random.default_rng(1912)
    arrays, meta = {}, {"generator": "tests/golden/make_golden_api.py", "numpy": np.__version__,
                        "columns": [], "xmajor": [], "rows": []}
    # --- fwht_column_in_place on every integer dtype ------------------------
    for dt in DTYPES:
        info = np.iinfo(dt)
        for k in (0, 1, 3, 6, 7, 10, 13):
            for kind in ("small", "full"):
                if kind == "small":
                    lo, hi = (0, 6) if info.min == 0 else (-5, 6)
                else:
                    lo, hi = info.min, info.max
                col = rng.integers(lo, hi, size=1 << k, dtype=dt, endpoint=(kind == "full"))
                if kind == "full" and k >= 3:
                    col[1] = info.min       # numpy abs(MIN) == MIN for signed dtypes
                    col[2] = info.max
                key = f"col_{dt}_{k}_{kind}"
                arrays[key + "_in"] = col.copy()
                with np.errstate(over="ignore"):
                    out, mx = se.fwht_column_in_place(col)
                arrays[key + "_out"] = out.copy()
                meta["columns"].append({"key": key, "dtype": dt, "k": k, "max_abs": int(mx)})
    # strided view: every 3rd element of a longer int16 vector, and a
    # negative-stride int32 view
    base = rng.integers(-100, 100, size=3 * 256, dtype=np.int16)
    arrays["strided_base_in"] = base.copy()
    _, mx = se.fwht_column_in_place(base[::3])
    arrays["strided_base_out"] = base.copy()
    meta["strided_max_abs"] = int(mx)
    neg = rng.integers(-100, 100, size=512, dtype=np.int32)
    arrays["neg_in"] = neg.copy()
    _, mx = se.fwht_column_in_place(neg[::-1])
    arrays["neg_out"] = neg.copy()
    meta["neg_max_abs"] = int(mx)
    # --- x-major polarity + transform ---------------------------------------
    for n, m, seed, bij in [(6, 5, 2, False), (8, 8, 0, True), (10, 7, 3, False), (12, 12, 0, True)]:
        s = se.generate_sbox(n, m, seed, bijective=bij)
        wt = sw_ref.build_polarity_xmajor(s)
        rec = {"n": n, "m": m, "seed": seed, "bijective": bij, "sha_polarity_xmajor": sha(wt)}
        sw_ref.transform_xmajor_in_place(wt)
        rec["sha_spectrum_xmajor"] = sha(wt)
        meta["xmajor"].append(rec)
    # --- transform_rows_in_place with maxima_out on int64 / int16 stores ------
    for dt, n, m, seed in [("int64", 7, 5, 1), ("int16", 6, 4, 2)]:
        s = se.generate_sbox(n, m, seed)
        rows = se.polarity_truth_table(s).rows.astype(dt)
        arrays[f"rows_{dt}_in"] = rows.copy()
        mo = np.zeros(rows.shape[0], dtype=np.int64)
        sw_ref.transform_rows_in_place(rows, maxima_out=mo)
        arrays[f"rows_{dt}_out"] = rows.copy()
        arrays[f"rows_{dt}_maxima"] = mo
        meta["rows"].append({"dtype": dt, "n": n, "m": m, "seed": seed})
    # --- column_nonlinearity -------------------------------------------------
    meta["column_nonlinearity"] = [[pw, mx, sw_ref.column_nonlinearity(pw, mx)]
                                   for pw, mx in [(256, 32), (65536, 1652), (16, 16), (1 << 20, 7586)]]
    np.savez_compressed(os.path.join(HERE, "golden_api.npz"), **arrays)
    with open(os.path.join(HERE, "golden_api.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(len(meta["columns"]), "columns;", meta["xmajor"])


if __name__ == "__main__":
    main()
