"""A/B of the multi-pass NL path: tensor-core pass A (default) vs the ALU pass A (SBW_TC=0)."""
import os, subprocess, sys, json
code = r'''
import sys, json, torch, numpy as np
sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw
res = {}
for (n, m, lo, hi) in [(17, 8, 1, 256), (20, 20, 1, 1 << 14), (24, 16, 1, 64), (18, 18, 1000, 3000)]:
    s = sw.generate_sbox(n, m, 0, bijective=False)
    mx, key = sw.component_max_abs_device(s, lo, hi)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); sw.component_max_abs_device(s, lo, hi); e1.record(); torch.cuda.synchronize()
    res[f"{n}x{m}"] = [mx.cpu().numpy().astype(np.int64).tolist(), int(key.item()), e0.elapsed_time(e1)]
print(json.dumps(res))
'''
out = {}
for tc in ("1", "0"):
    p = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, SBW_TC=tc), capture_output=True, text=True, timeout=600)
    if p.returncode: print(p.stderr[-2000:]); sys.exit(1)
    out[tc] = json.loads(p.stdout.strip().splitlines()[-1])
for k in out["1"]:
    a, b = out["1"][k], out["0"][k]
    print(k, "match" if a[:2] == b[:2] else "MISMATCH", f"tc {a[2]:.2f} ms  alu {b[2]:.2f} ms")
