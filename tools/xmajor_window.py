"""Experiment: x-major 16x16 slice as mask windows whose mask-major scratch
stays in L2 (sbw_spectrum layout 1 per window, output offset into the full
pitch) vs one call over the whole slice.  Checks the outputs are identical."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw
from paper_1912_03732_b200 import device as _dev

s = sw.generate_sbox(16, 16, 0, bijective=True)
lo, hi = 1, 1 << 14
rows = hi - lo
dev = torch.device("cuda:0")
lib = _dev.load_library()
tab = _dev.device_table(s, dev)
ref, _ = sw.spectrum_device(s, lo, hi, layout="x")
out = torch.empty_like(ref)
mx = torch.empty(rows, dtype=torch.int32, device=dev)
st = _dev.stream_handle(dev)


def run(W, scratch, nbytes):
    for v0 in range(lo, hi, W):
        v1 = min(hi, v0 + W)
        o = out.view(-1)[v0 - lo:]
        _dev.check(lib.sbw_spectrum(_dev.ptr(tab), _dev.table_bytes(s.m), 16, 16, v0, v1, 1, _dev.ptr(o), rows,
                                    _dev.ptr(mx[v0 - lo:]), _dev.ptr(scratch), nbytes, st))


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


t_full = timeit(lambda: sw.spectrum_device(s, lo, hi, layout="x", out=ref))
print(f"one call: {t_full:.3f} ms", flush=True)
for W in (64, 128, 192, 256, 296, 384, 444, 592, 888, 1184):
    nbytes = lib.sbw_spectrum_scratch_bytes(16, 16, lo, lo + W, 1)
    scratch = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    out.zero_()
    t = timeit(lambda: run(W, scratch, nbytes))
    ok = torch.equal(out, ref)
    print(f"W={W:5d} scratch {nbytes / 2**20:7.1f} MiB: {t:.3f} ms exact={ok}", flush=True)
    del scratch
