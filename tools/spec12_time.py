"""configs[1]: 12x12 materialised spectrum in both layouts + NL, device-resident (development helper)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw  # noqa: E402

s = sw.generate_sbox(12, 12, 0, bijective=True)
for layout in ("mask", "x"):
    out = None
    for _ in range(3):
        out, mx = sw.spectrum_device(s, 1, 1 << 12, layout=layout, out=out)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out, mx = sw.spectrum_device(s, 1, 1 << 12, layout=layout, out=out)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    gb = 4095 * 4096 * 4 / 1e9
    print(f"12x12 spectrum {layout}-major (4095 x 4096 int32 = {gb * 1e3:.0f} MB) + maxima: {best * 1e3:.1f} us, "
          f"{gb / best:.2f} TB/s written", flush=True)
