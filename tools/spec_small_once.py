"""Materialised spectra for n = 12..15 (m = n, seed 0) in both layouts, each
run twice -- for ncu launch lists of the spectrum kernels (development)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [12]:
    s = sw.generate_sbox(n, n, 0, bijective=True)
    for layout in ("mask", "x"):
        out = None
        for _ in range(2):
            out, mx = sw.spectrum_device(s, 1, 1 << n, layout=layout, out=out)
        torch.cuda.synchronize()
        print(n, layout, tuple(out.shape), int(mx.max()))
