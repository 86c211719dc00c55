"""A/B: overlapped (default) vs serialized (SBW_K3_SERIAL=1) K3 batches, full NL (development helper)."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw  # noqa: E402

for name, (n, m) in {"20x20": (20, 20), "24x16": (24, 16)}.items():
    s = sw.generate_sbox(n, m, 0, bijective=False)
    for rep in range(2):
        for serial in ("0", "1"):
            os.environ["SBW_K3_SERIAL"] = serial
            sw.component_max_abs_device(s)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            mx, key = sw.component_max_abs_device(s)
            e1.record()
            torch.cuda.synchronize()
            print(name, "serial" if serial == "1" else "overlap", f"{e0.elapsed_time(e1):.1f} ms", int(key.item()), flush=True)
