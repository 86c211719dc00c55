"""Wall time of the other 16x16 host-array producers (development helper)."""
import sys
import time

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw  # noqa: E402

s = sw.generate_sbox(16, 16, 0, bijective=True)
sw.fwht_transposed(s)  # one-time setup
for name, f in [("fwht_rowmajor", lambda: sw.fwht_rowmajor(s).rows),
                ("polarity_truth_table", lambda: sw.polarity_truth_table(s).rows),
                ("fwht_parallel(retain, 4 workers)", lambda: sw.fwht_parallel(s, workers=4)[0].rows)]:
    t0 = time.perf_counter()
    a = f()
    print(f"{name:34s} {time.perf_counter() - t0:7.3f} s ({a.nbytes / 1e9:.1f} GB)", flush=True)
    del a
