import sys, time
sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw
for n, m in [(20, 20), (24, 16)]:
    s = sw.generate_sbox(n, m, 0, bijective=False)
    r = sw.evaluate(s, method="fused", mode="stream")
    t0 = time.perf_counter()
    r = sw.evaluate(s, method="fused", mode="stream")
    t1 = time.perf_counter()
    r2 = sw.evaluate(s, method="parallel")
    t2 = time.perf_counter()
    print(f"{n}x{m}: evaluate(fused, stream) {t1 - t0:.3f} s, evaluate(parallel, retain default) {t2 - t1:.3f} s, NL {r.value} @ {r.argmin_v}", flush=True)
