"""Time the multi-pass (n >= 17) path on a mask subset (development helper)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw

name = sys.argv[1] if len(sys.argv) > 1 else "24x16"
masks = int(sys.argv[2]) if len(sys.argv) > 2 else 8
n, m, bij = {"20x20": (20, 20, False), "24x16": (24, 16, False)}[name]
s = sw.generate_sbox(n, m, 0, bijective=bij)
sw.component_max_abs_device(s, 1, 1 + masks)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
sw.component_max_abs_device(s, 1, 1 + masks)
e1.record()
torch.cuda.synchronize()
print(name, masks, e0.elapsed_time(e1), "ms")
