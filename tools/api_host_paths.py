"""Wall time of the numpy-facing API calls that move large arrays (development helper)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw  # noqa: E402

rng = np.random.default_rng(0)
rows = rng.integers(-3, 4, size=(4096, 1 << 16)).astype(np.int32)  # 1 GiB
col = rng.integers(-3, 4, size=1 << 24).astype(np.int32)
spec = sw.fwht_transposed(sw.generate_sbox(16, 16, 0, bijective=True))
for name, f in [("transform_rows_in_place 4096 x 2^16", lambda: sw.transform_rows_in_place(rows)),
                ("fwht_column_in_place 2^24", lambda: sw.fwht_column_in_place(col)),
                ("nonlinearity_from_spectrum 16x16 (17 GB)", lambda: sw.nonlinearity_from_spectrum(spec))]:
    f()
    t0 = time.perf_counter()
    f()
    print(f"{name:42s} {time.perf_counter() - t0:7.3f} s", flush=True)
