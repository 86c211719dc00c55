"""A/B check and timing of the n = 16 tensor-core path against the all-ALU tile
kernel (SBW_TC=0), both through component_max_abs_device (development helper).

python tools/tc_check.py          # runs both arms in subprocesses and compares
"""
import json
import os
import subprocess
import sys

import numpy as np

CASES = [  # (n, m, seed, bijective, v_lo, v_hi)
    (16, 16, 0, True, 1, None),
    (16, 16, 3, False, 1, None),
    (16, 16, 1, True, 300, 1000),
    (16, 16, 2, True, 1, 2),
    (16, 16, 2, True, 65000, 65536),
    (16, 8, 4, False, 1, None),
    (16, 12, 5, False, 7, 4000),
    (16, 20, 6, False, 1, 20000),
    (16, 16, 7, True, 1, 149),
]


def arm():
    import torch

    sys.path.insert(0, ".")
    import paper_1912_03732_b200 as sw

    out = {}
    for (n, m, seed, bij, lo, hi) in CASES:
        s = sw.generate_sbox(n, m, seed, bijective=bij)
        hi = hi or (1 << m)
        mx, key = sw.component_max_abs_device(s, lo, hi)
        out[str((n, m, seed, lo, hi))] = mx.cpu().numpy().astype(np.int64).tolist() + [int(key.item())]
    # timing of the full 16x16
    s = sw.generate_sbox(16, 16, 0, bijective=True)
    for _ in range(3):
        sw.component_max_abs_device(s, 1, 1 << 16)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(10):
        e0.record()
        sw.component_max_abs_device(s, 1, 1 << 16)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out["ms"] = best
    json.dump(out, sys.stdout)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "arm":
        arm()
        sys.exit(0)
    res = {}
    for tc in ("1", "0"):
        env = dict(os.environ, SBW_TC=tc)
        p = subprocess.run([sys.executable, __file__, "arm"], env=env, capture_output=True, text=True,
                           timeout=600)
        if p.returncode != 0:
            print(f"arm SBW_TC={tc} failed:\n{p.stderr[-3000:]}")
            sys.exit(1)
        res[tc] = json.loads(p.stdout.strip().splitlines()[-1])
    bad = 0
    for k in res["1"]:
        if k == "ms":
            continue
        a, b = np.array(res["1"][k]), np.array(res["0"][k])
        nd = int((a != b).sum())
        bad += nd
        print(f"{k}: {len(a)} comps, {nd} mismatches" + (f" first at {np.nonzero(a != b)[0][:5]}" if nd else ""))
    print(f"16x16 full NL: tc {res['1']['ms']:.3f} ms, alu {res['0']['ms']:.3f} ms")
    sys.exit(1 if bad else 0)
