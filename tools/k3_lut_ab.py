"""A/B of K3 pass A: k_tc_lut_emit (SBW_TC_LUT_EMIT=1) vs k_tc_hybrid<EMIT> (default): maxima on
several shapes must match; then full 20x20 / 24x16 times (argv: 'full')."""
import os, subprocess, sys, json
code = r'''
import sys, json, torch, numpy as np, hashlib
sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw
res = {}
full = len(sys.argv) > 1 and sys.argv[1] == "full"
cases = [(20, 20, 1, 1 << 20), (24, 16, 1, 1 << 16)] if full else [(17, 8, 1, 256), (20, 20, 1, 1 << 14), (24, 16, 1, 64), (18, 18, 1000, 3000), (19, 5, 1, 32), (21, 16, 7, 300), (22, 12, 1, 100), (23, 10, 1, 40)]
for (n, m, lo, hi) in cases:
    s = sw.generate_sbox(n, m, 0, bijective=False)
    mx, key = sw.component_max_abs_device(s, lo, hi)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3 if full else 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); sw.component_max_abs_device(s, lo, hi); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[f"{n}x{m}"] = [hashlib.sha256(mx.cpu().numpy().tobytes()).hexdigest()[:12], int(key.item()), best]
print(json.dumps(res))
'''
arg = sys.argv[1:2]
out = {}
for lut in ("1", "0"):
    p = subprocess.run(["timeout", "240", sys.executable, "-c", code] + arg, env=dict(os.environ, SBW_TC_LUT_EMIT=lut), capture_output=True, text=True)
    if p.returncode: print("rc", p.returncode, p.stderr[-1500:]); sys.exit(1)
    out[lut] = json.loads(p.stdout.strip().splitlines()[-1])
for k in out["1"]:
    a, b = out["1"][k], out["0"][k]
    print(k, "match" if a[:2] == b[:2] else "MISMATCH", f"lut {a[2]:.2f} ms  hybrid {b[2]:.2f} ms", a[0], b[0], flush=True)
