"""Sweep the K3 L2-ring knobs (SBW_K3_NA / SBW_K3_NB / SBW_K3_RING_L / SBW_K3_RING_R) on one
config and mask subset; prints device ms per setting (development helper).
usage: python tools/ring_sweep.py n m bijective masks "NA,L,R[,NB] NA,L,R ..." """
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw  # noqa: E402

n, m, bij, masks = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3] == "1", int(sys.argv[4])
settings = [tuple(int(x) for x in t.split(",")) for t in sys.argv[5].split()]
s = sw.generate_sbox(n, m, seed=0, bijective=bij)
v_hi = min(1 + masks, 1 << m)
ref = None
for st in settings:
    if st[0] == 0:
        os.environ["SBW_K3_RING"] = "0"
    else:
        os.environ["SBW_K3_RING"] = "1"
        os.environ["SBW_K3_NA"], os.environ["SBW_K3_RING_L"], os.environ["SBW_K3_RING_R"] = map(str, st[:3])
        os.environ["SBW_K3_NB"] = str(st[3]) if len(st) > 3 else "1000"
    sw.component_max_abs_device(s, 1, v_hi)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mx, key = sw.component_max_abs_device(s, 1, v_hi)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    h = mx.cpu().numpy()
    if ref is None:
        ref = h
    print(f"{n}x{m} masks {v_hi - 1} setting {st}: {best:.3f} ms  same={bool((h == ref).all())}", flush=True)
