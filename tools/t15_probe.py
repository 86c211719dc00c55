import sys, torch
sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw
s = sw.generate_sbox(15, 15, 0, bijective=True)
for _ in range(3): sw.component_max_abs_device(s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); sw.component_max_abs_device(s); e1.record(); torch.cuda.synchronize()
print("15x15 NL", e0.elapsed_time(e1), "ms")
