"""Full per-component max|W| of the 20x20 and 24x16 seed-0 boxes from the GPU into gpurun_out/ (to compare with tests/golden/_work chunks while the reference goldens are being generated)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw
for name, (n, m) in {"20x20": (20, 20), "24x16": (24, 16)}.items():
    s = sw.generate_sbox(n, m, 0, bijective=False)
    mx, key = sw.component_max_abs_device(s)
    np.save(f"gpurun_out/gpu_max_{name}.npy", mx.cpu().numpy())
    print(name, sw.walsh.decode_key(key, n))
