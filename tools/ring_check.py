"""A/B of the K3 L2 ring (SBW_K3_RING=1) against the batched path (=0):
bit-identical maxima + device time, on mask subsets (development helper).
usage: python tools/ring_check.py [n m bijective masks] ...  (default: a small set)"""
import hashlib
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw  # noqa: E402

cases = [(20, 20, False, 32768), (17, 17, True, 8192), (18, 12, False, 4095), (19, 16, False, 8192),
         (21, 16, False, 4096), (20, 20, False, 1 << 20 - 1)]
if len(sys.argv) > 1:
    a = sys.argv[1:]
    cases = [(int(a[i]), int(a[i + 1]), a[i + 2] == "1", int(a[i + 3])) for i in range(0, len(a), 4)]


def run(s, v_hi, ring):
    os.environ["SBW_K3_RING"] = "1" if ring else "0"
    sw.component_max_abs_device(s, 1, v_hi)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    mx, key = sw.component_max_abs_device(s, 1, v_hi)
    e1.record()
    torch.cuda.synchronize()
    return mx.cpu().numpy(), int(key.item()), e0.elapsed_time(e1)


for n, m, bij, masks in cases:
    s = sw.generate_sbox(n, m, seed=0, bijective=bij)
    v_hi = min(1 + masks, 1 << m)
    a_mx, a_key, a_ms = run(s, v_hi, False)
    b_mx, b_key, b_ms = run(s, v_hi, True)
    same = bool((a_mx == b_mx).all()) and a_key == b_key
    h = hashlib.sha256(b_mx.tobytes()).hexdigest()[:12]
    print(f"{n}x{m} masks {v_hi - 1}: batched {a_ms:.3f} ms, ring {b_ms:.3f} ms ({a_ms / b_ms:.2f}x) "
          f"identical={same} hash={h} min={b_mx.min()}", flush=True)
