"""Full-range x-major store of a bijective box: inverse path (default) vs the
mask-major + flat-transpose path (SBW_XMAJOR_INVERSE=0), device time by CUDA
events through spectrum_device(layout="x"), plus the inverse kernel alone."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw
from paper_1912_03732_b200 import device as dv
from paper_1912_03732_b200 import walsh


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for n in [int(x) for x in (sys.argv[1:] or ["12", "14", "16"])]:
    s = sw.generate_sbox(n, n, 0, bijective=True)
    gb = (1 << n) * ((1 << n) - 1) * 4 / 1e9
    out = torch.empty((1 << n, (1 << n) - 1), dtype=torch.int32, device="cuda:0")
    t_inv = timeit(lambda: sw.spectrum_device(s, layout="x", out=out))
    ref = out.clone()
    inv = walsh._inverse_if_bijective(s)
    lib = dv.load_library()
    dev = torch.device("cuda:0")
    itab = dv.device_table(inv, dev)
    nb = lib.sbw_xmajor_inverse_scratch_bytes(n, 1, 1 << n)
    scr = torch.empty(nb, dtype=torch.uint8, device=dev)
    st = dv.stream_handle(dev)
    t_kernel = timeit(lambda: dv.check(lib.sbw_xmajor_from_inverse(
        dv.ptr(itab), dv.table_bytes(n), n, 1, 1 << n, dv.ptr(out) + 4 * out.stride(0), out.stride(0),
        dv.ptr(scr), nb, st)))
    t_nl = timeit(lambda: sw.component_max_abs_device(s))
    os.environ["SBW_XMAJOR_INVERSE"] = "0"
    if n <= 15 or torch.cuda.get_device_properties(0).total_memory > 60 << 30:
        t_tr = timeit(lambda: sw.spectrum_device(s, layout="x", out=out), reps=3)
        same = torch.equal(out, ref)
    else:
        t_tr, same = float("nan"), None
    del os.environ["SBW_XMAJOR_INVERSE"]
    print(f"n={n} x-major full {gb:.3f} GB: inverse path {t_inv:.3f} ms (x-major kernel {t_kernel:.3f} ms = "
          f"{gb / t_kernel:.2f} TB/s, maxima {t_nl:.3f} ms); transpose path {t_tr:.3f} ms; identical={same}",
          flush=True)
    del out, ref, scr
    torch.cuda.empty_cache()
