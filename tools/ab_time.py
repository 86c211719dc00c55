"""Time 16x16 full NL for each libsbw variant in build_variants/ (one subprocess each)."""
import glob
import os
import subprocess
import sys

code = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw
n, m = int(sys.argv[1]), int(sys.argv[2])
s = sw.generate_sbox(n, m, 0, bijective=(n == m))
ref = None
for _ in range(3): mx, key = sw.component_max_abs_device(s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(10):
    e0.record(); sw.component_max_abs_device(s); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
import hashlib
h = hashlib.sha256(mx.cpu().numpy().tobytes()).hexdigest()[:12]
print(f"{best:.4f} {int(key.item())} {h}")
'''
n, m = (sys.argv[1], sys.argv[2]) if len(sys.argv) > 2 else ("16", "16")
for lib in sorted(glob.glob("build_variants/libsbw_*.so")) + ["paper_1912_03732_b200/libsbw.so"]:
    env = dict(os.environ, SBW_LIB_PATH=os.path.abspath(lib))
    p = subprocess.run([sys.executable, "-c", code, n, m], env=env, capture_output=True, text=True, timeout=300)
    print(f"{os.path.basename(lib):28s} {p.stdout.strip() or p.stderr.strip()[-300:]}")
