"""Quick device timing of the fused NL kernels (development helper)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw
from paper_1912_03732_b200 import device as d


def time_nl(s, reps=5, lo=1, hi=None):
    hi = hi or (1 << s.m)
    for _ in range(2):
        sw.component_max_abs_device(s, lo, hi)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        e0.record()
        sw.component_max_abs_device(s, lo, hi)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


if __name__ == "__main__":
    peak = d.ctypes.c_double(0)
    ms = d.ctypes.c_double(0)
    d.check(d.load_library().sbw_int32_peak(d.ctypes.byref(peak), d.ctypes.byref(ms), None))
    print(f"int32 peak {peak.value/1e12:.2f} Tops/s ({ms.value:.2f} ms)")
    print(d.device_info(0))
    for (n, m, bij, lo, hi) in [(8, 8, True, 1, None), (12, 12, True, 1, None), (16, 16, True, 1, None),
                                (20, 20, False, 1, 1 << 14), (24, 16, False, 1, 64)]:
        s = sw.generate_sbox(n, m, 0, bijective=bij)
        t = time_nl(s, lo=lo, hi=hi)
        nv = (hi or (1 << m)) - lo
        coeff = nv * (1 << n)
        ops = n * (1 << n) * nv
        print(f"{n}x{m} masks={nv}: {t:.3f} ms  {coeff/t/1e9:.3f} Tcoeff/s  {ops/t/1e9:.2f} Tops/s"
              f"  frac={ops/t/1e9*1e12/peak.value:.3f}")
