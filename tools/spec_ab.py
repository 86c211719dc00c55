"""Mask-major 16x16 spectrum slice (16383 rows, 4.3 GB) for each libsbw variant in
build_variants/ (one subprocess each, SBW_LIB_PATH), best of 5, with a sha of the maxima."""
import glob
import os
import subprocess
import sys

code = r'''
import sys, torch, hashlib
sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw
s = sw.generate_sbox(16, 16, 0, bijective=True)
out = None
for _ in range(2): out, mx = sw.spectrum_device(s, 1, 1 << 14, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(5):
    e0.record(); out, mx = sw.spectrum_device(s, 1, 1 << 14, out=out); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
h = hashlib.sha256(out[::997].cpu().numpy().tobytes()).hexdigest()[:12]
print(f"{best:.4f} ms {16383 * 65536 * 4 / best / 1e9:.2f} TB/s {h}")
'''
for lib in sorted(glob.glob("build_variants/libsbw_*.so")) + ["paper_1912_03732_b200/libsbw.so"]:
    env = dict(os.environ, SBW_LIB_PATH=os.path.abspath(lib))
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    print(f"{os.path.basename(lib):28s} {p.stdout.strip() or p.stderr.strip()[-300:]}")
