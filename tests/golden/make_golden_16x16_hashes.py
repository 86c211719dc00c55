"""sha256 of the full 16x16 (seed 0) Walsh matrix in both layouts, computed by
the REFERENCE (build container only; ~16 GiB of RAM, ~5 min).

  mask-major: sha256 of fwht_fused(s, "retain")[0].rows (walsh.py:204-248),
              the (2^16 - 1) x 2^16 int32 C-order array, in one pass;
  x-major:    sha256 of the bytes of rows.T in C order (= the reference's
              x-major store wt[x][v-1], walsh.py:117-131 / :174), fed in
              blocks of 1024 x-rows (rows[:, a:a+1024].T contiguous), which is
              the same byte stream as hashing rows.T contiguous at once.

Writes tests/golden/hashes_16x16.json.  Run:
  PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_16x16_hashes.py
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import sboxeval as se  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    t0 = time.time()
    s = se.generate_sbox(16, 16, 0, bijective=True)
    spec, cm = se.fwht_fused(s, mode="retain")
    rows = spec.rows
    t1 = time.time()
    hm = hashlib.sha256()
    for a in range(0, rows.shape[0], 1024):
        hm.update(np.ascontiguousarray(rows[a:a + 1024]).tobytes())
    hx = hashlib.sha256()
    for a in range(0, rows.shape[1], 1024):
        hx.update(np.ascontiguousarray(rows[:, a:a + 1024].T).tobytes())
    out = {"generator": "tests/golden/make_golden_16x16_hashes.py", "numpy": np.__version__,
           "config": "16x16 bijective seed 0", "shape_mask_major": list(rows.shape),
           "sha256_mask_major": hm.hexdigest(), "sha256_x_major": hx.hexdigest(),
           "nl": int(se.nonlinearity_from_maxima(cm).value),
           "argmin_v": int(se.nonlinearity_from_maxima(cm).argmin_v),
           "ref_transform_s": round(t1 - t0, 1)}
    with open(os.path.join(HERE, "hashes_16x16.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
