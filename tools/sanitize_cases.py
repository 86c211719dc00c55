"""Small end-to-end cases for compute-sanitizer (one tool per run)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw

for n, m in [(3, 4), (7, 5), (9, 9), (12, 6), (16, 3), (17, 2), (21, 2)]:
    s = sw.generate_sbox(n, m, seed=n + m)
    _, cm = sw.fwht_fused(s, mode="stream")
    if (1 << m) * (1 << n) <= 1 << 22:
        spec, cm2 = sw.fwht_fused(s, mode="retain")
        assert np.array_equal(cm.values, cm2.values)
        xm, _ = sw.spectrum_device(s, layout="x")
col = np.arange(1 << 10, dtype=np.int32)
sw.fwht_column_in_place(col)
sw.nonlinearity_bruteforce(sw.aes_sbox())
sw.walsh_direct(sw.aes_sbox(), 3, 7)
print("sanitize cases ok")
