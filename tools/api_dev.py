import sys, time
import torch
sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw
s = sw.generate_sbox(16, 16, 0, bijective=True)
for _ in range(3): sw.component_max_abs_device(s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter(); e0.record()
for _ in range(20): sw.component_max_abs_device(s)
e1.record(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"host enqueue {(t1 - t0) / 20 * 1e3:.3f} ms/call, wall {(t2 - t0) / 20 * 1e3:.3f} ms/call, device {e0.elapsed_time(e1) / 20:.3f} ms/call")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(20): sw.component_max_abs_device(s)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(8)
