"""Wall time of the 16x16 materialised-spectrum API calls (16 GiB to host)."""
import sys
import time

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw  # noqa: E402

s = sw.generate_sbox(16, 16, 0, bijective=True)
for name, f in [("fwht_transposed (first call)", lambda: sw.fwht_transposed(s)),
                ("fwht_transposed", lambda: sw.fwht_transposed(s)),
                ("fwht_fused(retain)", lambda: sw.fwht_fused(s, mode="retain")[0])]:
    t0 = time.perf_counter()
    w = f()
    t1 = time.perf_counter()
    gb = w.rows.nbytes / 1e9
    print(f"{name:30s} {t1 - t0:7.3f} s  ({gb:.1f} GB to host, {gb / (t1 - t0):.1f} GB/s)", flush=True)
    del w
