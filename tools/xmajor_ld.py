"""x-major spectrum into a pitch of 2^m - 1 (the reference's dense layout) vs a
padded, 16-byte aligned pitch (development helper)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw  # noqa: E402
from paper_1912_03732_b200 import device as d  # noqa: E402

lib = d.load_library()
dev = torch.device("cuda", 0)
s = sw.generate_sbox(16, 16, 0, bijective=True)
tab = d.device_table(s, dev)
lo, hi = 1, 1 << 14
st = torch.cuda.current_stream().cuda_stream
sb = lib.sbw_spectrum_scratch_bytes(16, 16, lo, hi, 1)
scratch = torch.empty(sb, dtype=torch.uint8, device=dev)
for ld in (hi - lo, hi - lo + 1, 16384 + 32):
    out = torch.empty((1 << 16) * ld, dtype=torch.int32, device=dev)
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.check(lib.sbw_spectrum(d.ptr(tab), d.table_bytes(16), 16, 16, lo, hi, 1, out.data_ptr(), ld, None,
                                 scratch.data_ptr(), sb, st))
        e1.record()
        torch.cuda.synchronize()
    print(f"x-major ld {ld}: {e0.elapsed_time(e1):.2f} ms", flush=True)
    del out
