import sys, torch
sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw
s = sw.generate_sbox(16, 16, 0, bijective=True)
for layout in ("mask", "x"):
    lo, hi = 1, 1 << 14  # 16383 rows = 4 GiB
    out = None
    for _ in range(2):
        out, mx = sw.spectrum_device(s, lo, hi, layout=layout, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); out, mx = sw.spectrum_device(s, lo, hi, layout=layout, out=out); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    gb = (hi - lo) * 65536 * 4 / 1e9
    print(f"spectrum {layout}-major 16x16 rows {hi-lo}: {ms:.2f} ms, {gb:.2f} GB written, {gb/ms:.2f} TB/s")
    del out
    torch.cuda.empty_cache()
