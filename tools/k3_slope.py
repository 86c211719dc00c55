import sys, time
import torch
sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw
name = sys.argv[1]
n, m, bij = {"20x20": (20, 20, False), "24x16": (24, 16, False)}[name]
s = sw.generate_sbox(n, m, 0, bijective=bij)
for k in [1, 2, 4, 8, 16, 32, 64]:
    sw.component_max_abs_device(s, 1, 1 + k); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    sw.component_max_abs_device(s, 1, 1 + k)
    e1.record(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(name, k, f"gpu {e0.elapsed_time(e1):.3f} ms  host-enqueue {1e3*(t1-t0):.3f} ms  wall {1e3*(t2-t0):.3f}")
