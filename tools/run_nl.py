"""Run one full-range NL evaluation (profiling driver): python tools/run_nl.py N M [reps]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw

n, m = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
s = sw.generate_sbox(n, m, 0, bijective=(n == m))
for _ in range(reps):
    mx, key = sw.component_max_abs_device(s)
torch.cuda.synchronize()
print("key", int(key.item()))
