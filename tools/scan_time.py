"""Device throughput of the spectrum-scan reducer (sbw_row_maxabs: nonlinearity_from_spectrum on a
device-resident spectrum) against the HBM copy roofline (development helper)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1912_03732_b200 import device as d  # noqa: E402

lib = d.load_library()
dev = torch.device("cuda", 0)
hbm = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6552.3) if os.path.exists("MEASURED_PEAKS.json") else 6552.3
st = torch.cuda.current_stream().cuda_stream
for rows, cols in [(16383, 65536), (4095, 4096), (65535, 4096)]:
    x = torch.randint(-1000, 1000, (rows, cols), dtype=torch.int32, device=dev)
    rm = torch.empty(rows, dtype=torch.int64, device=dev)
    key = torch.zeros(1, dtype=torch.int64, device=dev)
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.check(lib.sbw_row_maxabs(x.data_ptr(), rows, cols, cols, rm.data_ptr(), key.data_ptr(), st))
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    nb = rows * cols * 4
    print(f"scan {rows} x {cols}: {best:.3f} ms, {nb / best / 1e6:.0f} GB/s = {nb / best / 1e6 / hbm:.2f} of HBM", flush=True)
    del x
