"""A/B of the n = 16 NL kernels: k_tc_lut (SBW_TC_LUT=1, default) vs k_tc_hybrid<NL,16>
(SBW_TC_LUT=0): full 16x16 maxima hash, key and best-of-10 device time, one subprocess each."""
import os
import subprocess
import sys

code = r'''
import sys, torch, hashlib
sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw
s = sw.generate_sbox(16, 16, 0, bijective=True)
for _ in range(3): mx, key = sw.component_max_abs_device(s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(10):
    e0.record(); sw.component_max_abs_device(s); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
h = hashlib.sha256(mx.cpu().numpy().tobytes()).hexdigest()[:12]
mx2, _ = sw.component_max_abs_device(s, 1000, 1003)
print(f"best {min(ts):.4f} median {sorted(ts)[5]:.4f} key {int(key.item())} sha {h} max {int(mx.max())} first {mx[:4].tolist()} slice {mx2.tolist()}")
'''
for lut in ("1", "0", "1", "0"):
    env = dict(os.environ, SBW_TC_LUT=lut)
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    print(f"SBW_TC_LUT={lut}: {p.stdout.strip() or p.stderr.strip()[-600:]}", flush=True)
