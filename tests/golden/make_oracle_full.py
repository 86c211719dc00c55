"""Every per-component max|W| of the two large configs, from the compiled ORACLE.

BASELINE.json configs[3] (20x20) and configs[4] (24x16), seed 0, non-bijective,
all masks v = 1 .. 2^m - 1, through oracle/sbw_oracle.c (the C restatement of
the reference's stream body, walsh.py:237-240).  The arrays are committed so the
GPU tests can compare the device's full output element for element without
re-running ~5 core-hours of CPU work on the GPU box.

Provenance chain (all checked by tests/test_oracle.py on the CPU):
  * the C oracle equals the reference's full 16x16 maxima (golden_arrays.npz),
    its sampled 20x20 / 24x16 masks (golden.json), and
  * every chunk of the reference's OWN full run present under
    tests/golden/full_work/ (tests/golden/make_golden_full.py), and the final
    full_<name>.npz once that run has finished.

Run (any host with gcc; a few minutes on 8 cores):
    make -C oracle && python tests/golden/make_oracle_full.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import sbw_oracle as orc  # noqa: E402

CONFIGS = {"20x20": (20, 20), "24x16": (24, 16)}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def main():
    summary = {"generator": "tests/golden/make_oracle_full.py (oracle/sbw_oracle.c)", "configs": {}}
    for name, (n, m) in CONFIGS.items():
        t = orc.gen_table(n, m, 0, False)
        t0 = time.time()
        mx = orc.component_max_abs_c(t, n, 1, 1 << m)
        dt = time.time() - t0
        assert mx.max() < (1 << 16)
        values = ((1 << n) - mx) >> 1
        idx = int(np.argmin(values))
        summary["configs"][name] = {
            "n": n, "m": m, "seed": 0, "bijective": False,
            "nl": int(values[idx]), "argmin_v": idx + 1, "max_abs": int(mx.max()),
            "sha_maxima_i64": sha(values.astype(np.int64)),
            "sha_max_abs_u16": sha(mx.astype(np.uint16)),
            "seconds": round(dt, 1), "threads": os.cpu_count(),
        }
        np.savez_compressed(os.path.join(HERE, f"oracle_full_{name}.npz"), max_abs=mx.astype(np.uint16))
        print(name, summary["configs"][name], flush=True)
    with open(os.path.join(HERE, "oracle_full.json"), "w") as f:
        json.dump(summary, f, indent=1)


if __name__ == "__main__":
    main()
