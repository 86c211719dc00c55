"""A/B of the n = 11..15 tensor-core NL path (default) vs the tile kernel (SBW_TC=0)."""
import json
import os
import subprocess
import sys

code = r'''
import sys, json, torch, numpy as np
sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw
res = {}
for (n, m, lo, hi) in [(15, 15, 1, 1 << 15), (14, 14, 1, 1 << 14), (13, 13, 1, 1 << 13), (12, 12, 1, 1 << 12),
                       (11, 11, 1, 1 << 11), (12, 16, 3, 5000), (15, 1, 1, 2), (11, 5, 1, 32), (13, 9, 100, 300),
                       (14, 20, 70000, 71000)]:
    s = sw.generate_sbox(n, m, 7, bijective=(n == m))
    mx, key = sw.component_max_abs_device(s, lo, hi)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); sw.component_max_abs_device(s, lo, hi); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[f"{n}x{m} [{lo},{hi})"] = [mx.cpu().numpy().astype(np.int64).tolist(), int(key.item()), best]
print(json.dumps(res))
'''
out = {}
for tc in ("1", "0"):
    p = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, SBW_TC=tc), capture_output=True,
                       text=True, timeout=600)
    if p.returncode:
        print(p.stderr[-3000:])
        sys.exit(1)
    out[tc] = json.loads(p.stdout.strip().splitlines()[-1])
bad = 0
for k in out["1"]:
    a, b = out["1"][k], out["0"][k]
    ok = a[:2] == b[:2]
    bad += not ok
    print(f"{k:22s} {'match' if ok else 'MISMATCH'}  tc {a[2]:.3f} ms  alu {b[2]:.3f} ms")
sys.exit(1 if bad else 0)
