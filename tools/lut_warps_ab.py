"""A/B of k_tc_lut (8 transform warps) vs k_tc_lut16 (SBW_LUT_WARPS=16) and k_tc_hybrid (SBW_TC_LUT=0)."""
import os, subprocess, sys
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
i16 = sw.identity_sbox(16)
mi, ki = sw.component_max_abs_device(i16, 1, 300)
print(f"best {min(ts):.4f} median {sorted(ts)[5]:.4f} key {int(key.item())} sha {h} slice {mx2.tolist()} ident {int(mi.min())} {int(mi.max())}")
'''
for env in ({"SBW_LUT_WARPS": "16"}, {"SBW_LUT_WARPS": "8"}, {"SBW_TC_LUT": "0"}, {"SBW_LUT_WARPS": "16"}, {"SBW_LUT_WARPS": "8"}):
    p = subprocess.run(["timeout", "120", sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True)
    print(f"{env}: {p.stdout.strip() or p.stderr.strip()[-600:]}", flush=True)
