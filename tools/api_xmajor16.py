"""Wall time of the full 16x16 x-major export to a host array (17.2 GB):
inverse path (row chunks) vs SBW_XMAJOR_INVERSE=0 (mask chunks + transpose)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw  # noqa: E402

s = sw.generate_sbox(16, 16, 0, bijective=True)
out = np.empty((65536, 65535), dtype=np.int32)
for env in ("1", "1", "0"):
    os.environ["SBW_XMAJOR_INVERSE"] = env
    t0 = time.perf_counter()
    sw.spectrum_to_host(s, layout="x", out=out)
    dt = time.perf_counter() - t0
    print(f"SBW_XMAJOR_INVERSE={env}: {dt:.3f} s ({out.nbytes / 1e9 / dt:.1f} GB/s)", flush=True)
