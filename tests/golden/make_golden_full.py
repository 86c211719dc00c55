"""Full per-component maxima of the two large configs, computed by the REFERENCE.

BASELINE.json configs[3] (20x20, non-bijective, seed 0) and configs[4]
(24x16, non-bijective, seed 0) are too large for the reference's own
``fwht_fused(mode="stream")`` in one process (~15 core-hours each), so this
script runs exactly the reference's stream body over every mask

    polarity_row(s, v, out=buf)                 pkg/src/sboxeval/sbox.py:145-152
    _, max_abs = fwht_column_in_place(buf)      pkg/src/sboxeval/walsh.py:73-104
    maxima[v-1] = column_nonlinearity(pw, max_abs)   walsh.py:107-114

(the loop at pkg/src/sboxeval/walsh.py:237-240), with the masks split into
contiguous chunks over a multiprocessing pool, the way ``fwht_parallel``
splits them (pkg/src/sboxeval/parallel.py:38-57).  The table is the
reference's own ``generate_sbox`` (sbox.py:102-111).  Chunks are checkpointed
under ``tests/golden/full_work/`` (committed as they finish, gpurun-ignored) so a run can resume
in a new container.

Output (committed): ``tests/golden/full_<name>.npz`` holding ``max_abs``
(uint16, one entry per component v = 1..2^m-1; every value < 2^15 here) and
``tests/golden/full_maxima.json`` with the sha256 prefix of the int64
``ColumnMaxima.values`` (= per-component NL) and the overall NL / argmin_v.

Run (build container only; reads /root/reference):
    PYTHONDONTWRITEBYTECODE=1 nice -n 19 python tests/golden/make_golden_full.py [procs [rev]]
    python tests/golden/make_golden_full.py finalize     # assemble whatever configs are complete
"""
from __future__ import annotations

import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
WORK = os.path.join(HERE, "full_work")

CONFIGS = {"20x20": (20, 20, 4096), "24x16": (24, 16, 256)}  # n, m, masks per chunk

_S = {}


def _sbox(name):
    if name not in _S:
        sys.path.insert(0, REF)
        import sboxeval as se
        import sboxeval.walsh as sw
        se.column_nonlinearity = sw.column_nonlinearity
        n, m, _ = CONFIGS[name]
        _S[name] = (se, se.generate_sbox(n, m, seed=0, bijective=False))
    return _S[name]


def _chunk(args):
    name, lo, hi = args
    path = os.path.join(WORK, f"{name}_{lo:08d}_{hi:08d}.npy")
    if os.path.exists(path):
        return name, lo, hi, 0.0
    se, s = _sbox(name)
    t0 = time.time()
    buf = np.empty(1 << s.n, dtype=np.int32)
    out = np.empty(hi - lo, dtype=np.uint16)
    for v in range(lo, hi):
        se.polarity_row(s, v, out=buf)
        _, max_abs = se.fwht_column_in_place(buf)
        se.column_nonlinearity(1 << s.n, max_abs)  # parity check, as the reference does
        out[v - lo] = max_abs
    np.save(path + ".tmp.npy", out)
    os.replace(path + ".tmp.npy", path)
    return name, lo, hi, time.time() - t0


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def main():
    procs = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    os.makedirs(WORK, exist_ok=True)
    jobs = []
    for name, (n, m, step) in CONFIGS.items():
        total = (1 << m)
        jobs += [(name, lo, min(lo + step, total)) for lo in range(1, total, step)]
    # one config at a time (20x20 first, the cheaper one), so a run cut short
    # still leaves one config complete
    order = sys.argv[3].split(",") if len(sys.argv) > 3 else list(CONFIGS)
    jobs.sort(key=lambda j: (order.index(j[0]), j[1]))
    if len(sys.argv) > 2 and sys.argv[2] == "rev":  # a second runner from the other end
        jobs.reverse()
    t0 = time.time()
    with mp.Pool(procs) as pool:
        for k, (name, lo, hi, dt) in enumerate(pool.imap_unordered(_chunk, jobs)):
            print(f"[{time.time() - t0:8.0f}s] {k + 1}/{len(jobs)} {name} {lo}..{hi} {dt:.1f}s",
                  flush=True)
    finalize()


def finalize():
    """Assemble tests/golden/full_<name>.npz and full_maxima.json for every
    config whose chunks are all present (a run cut short still pins what it
    finished; the other config keeps its per-chunk checks)."""
    summary = {"generator": "tests/golden/make_golden_full.py", "numpy": np.__version__,
               "configs": {}}
    for name, (n, m, step) in CONFIGS.items():
        paths = [os.path.join(WORK, f"{name}_{lo:08d}_{min(lo + step, 1 << m):08d}.npy")
                 for lo in range(1, 1 << m, step)]
        missing = [q for q in paths if not os.path.exists(q)]
        if missing:
            print(f"{name}: {len(paths) - len(missing)}/{len(paths)} chunks, not finalised", flush=True)
            continue
        max_abs = np.concatenate([np.load(q) for q in paths])
        assert max_abs.shape[0] == (1 << m) - 1
        values = ((1 << n) - max_abs.astype(np.int64)) >> 1  # ColumnMaxima.values
        idx = int(np.argmin(values))
        summary["configs"][name] = {
            "n": n, "m": m, "seed": 0, "bijective": False,
            "nl": int(values[idx]), "argmin_v": idx + 1, "max_abs": int(max_abs.max()),
            "sha_maxima_i64": sha(values.astype(np.int64)),
            "sha_max_abs_u16": sha(max_abs),
        }
        np.savez_compressed(os.path.join(HERE, f"full_{name}.npz"), max_abs=max_abs)
    if summary["configs"]:
        with open(os.path.join(HERE, "full_maxima.json"), "w") as f:
            json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "finalize":
        finalize()
    else:
        main()
