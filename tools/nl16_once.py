"""Run the 16x16 full NL twice (warm-up + one more) for ncu captures:
  ncu --set full -k regex:k_tc --launch-skip 1 --launch-count 1 -o X python tools/nl16_once.py"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw  # noqa: E402

s = sw.generate_sbox(16, 16, 0, bijective=True)
for _ in range(2):
    mx, key = sw.component_max_abs_device(s)
torch.cuda.synchronize()
print(sw.walsh.decode_key(key, 16))
