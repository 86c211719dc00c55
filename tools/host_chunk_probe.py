"""spectrum_to_host(16x16, all 65535 masks, 17.2 GB) wall time in a fresh
process for one chunk size (first call = pinned staging allocation
included), then a second call: python tools/host_chunk_probe.py CHUNK_MIB"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw  # noqa: E402

mib = int(sys.argv[1])
s = sw.generate_sbox(16, 16, 0, bijective=True)
sw.component_max_abs_device(s, 1, 3)  # context, library, table upload
torch.cuda.synchronize()
for call in ("first", "second"):
    t0 = time.perf_counter()
    out, mx = sw.spectrum_to_host(s, chunk_bytes=mib << 20)
    t1 = time.perf_counter()
    print(f"chunk {mib} MiB {call}: {t1 - t0:.3f} s = {out.nbytes / (t1 - t0) / 1e9:.1f} GB/s", flush=True)
    del out
