"""One 16x16 mask-major spectrum slice (16383 masks, 4.3 GB) after a warm-up
call: the ncu target for the staged spectrum epilogue."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw  # noqa: E402

s = sw.generate_sbox(16, 16, 0, bijective=True)
out, mx = sw.spectrum_device(s, 1, 1 << 14)
out, mx = sw.spectrum_device(s, 1, 1 << 14, out=out)
torch.cuda.synchronize()
print("ok", int(mx.max()))
