"""Device throughput of the generic in-place FWHT (sbw_fwht_inplace, the
fwht_column_in_place / transform_rows_in_place kernel) on device-resident
int32 rows, against the HBM copy roofline (development helper)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1912_03732_b200 import device as d  # noqa: E402

lib = d.load_library()
dev = torch.device("cuda", 0)
peaks = json.load(open("MEASURED_PEAKS.json")) if os.path.exists("MEASURED_PEAKS.json") else {}
hbm = peaks.get("hbm_gbs", 6552.3)
st = torch.cuda.current_stream().cuda_stream
for count, k in [(4095, 12), (65535, 12), (1024, 16), (16384, 16), (64, 20), (4, 24), (64, 24)]:
    x = torch.randint(-5, 6, (count, 1 << k), dtype=torch.int32, device=dev)
    mx = torch.empty(count, dtype=torch.int64, device=dev)
    d.check(lib.sbw_fwht_inplace(x.data_ptr(), k, count, mx.data_ptr(), st))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record()
        d.check(lib.sbw_fwht_inplace(x.data_ptr(), k, count, mx.data_ptr(), st))
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    nbytes = count * (1 << k) * 4
    passes = 1 + max(0, -(-(k - 12) // 6)) if k >= 12 else -(-k // 6)
    print(f"count {count:6d} k {k:2d}: {best:8.3f} ms, {2 * nbytes / best / 1e6:7.0f} GB/s per pass-equivalent "
          f"(1 read + 1 write of {nbytes / 1e6:.0f} MB), {passes} passes -> "
          f"{passes * 2 * nbytes / best / 1e6:7.0f} GB/s moved = {passes * 2 * nbytes / best / 1e6 / hbm:.2f} of HBM",
          flush=True)
    del x
