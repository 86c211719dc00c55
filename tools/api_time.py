"""Wall time of the drop-in Python API calls for 16x16 (what a sboxeval user sees)."""
import sys
import time

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw  # noqa: E402

s = sw.generate_sbox(16, 16, 0, bijective=True)
for name, f in [("fwht_fused(stream)", lambda: sw.fwht_fused(s, mode="stream")),
                ("evaluate(method=fused)", lambda: sw.evaluate(s, method="fused")),
                ("evaluate(method=parallel, stream)", lambda: sw.evaluate(s, method="parallel", mode="stream")),
                ("component_max_abs_device", lambda: sw.component_max_abs_device(s))]:
    for _ in range(3):
        f()
    t0 = time.perf_counter()
    for _ in range(10):
        r = f()
    if name == "component_max_abs_device":
        import torch
        torch.cuda.synchronize()
    print(f"{name:36s} {(time.perf_counter() - t0) / 10 * 1e3:8.3f} ms per call", flush=True)
