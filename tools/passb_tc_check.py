"""Quick check of the tensor-core pass B (n = 22..24) against the oracle and the
fp32 pass B (SBW_PASSB_TC=0), with timing: python tools/passb_tc_check.py"""
import os, subprocess, sys, json
code = r'''
import sys, json, torch, numpy as np
sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw
res = {}
for (n, m, lo, hi) in [(17, 8, 1, 256), (18, 6, 1, 64), (19, 6, 1, 64), (20, 8, 1, 256), (21, 6, 1, 64),
                       (22, 6, 1, 64), (23, 5, 1, 32), (24, 4, 1, 16), (24, 16, 1000, 1064)]:
    s = sw.generate_sbox(n, m, 0, bijective=False)
    mx, key = sw.component_max_abs_device(s, lo, hi)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); sw.component_max_abs_device(s, lo, hi); e1.record(); torch.cuda.synchronize()
    res[f"{n}x{m}:{lo}-{hi}"] = [mx.cpu().numpy().astype(np.int64).tolist(), int(key.item()), e0.elapsed_time(e1)]
print(json.dumps(res))
'''
out = {}
for tc in ("1", "0"):
    p = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, SBW_PASSB_TC=tc), capture_output=True,
                       text=True, timeout=300)
    if p.returncode:
        print(p.stderr[-3000:]); sys.exit(1)
    out[tc] = json.loads(p.stdout.strip().splitlines()[-1])
bad = 0
for k in out["1"]:
    a, b = out["1"][k], out["0"][k]
    ok = a[:2] == b[:2]
    bad += not ok
    print(k, "match" if ok else "MISMATCH", f"tc {a[2]:.2f} ms  fp32 {b[2]:.2f} ms")
    if not ok:
        print("  tc  ", a[0][:8], a[1]); print("  fp32", b[0][:8], b[1])
sys.exit(1 if bad else 0)
