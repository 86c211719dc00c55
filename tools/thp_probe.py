import mmap, time, numpy as np, torch
n = 2 << 30
p = torch.empty((n // 4,), dtype=torch.int32, pin_memory=True); p.fill_(3)
for mode in ("np.empty", "mmap+THP", "mmap"):
    if mode == "np.empty":
        b = np.empty(n // 4, dtype=np.int32)
    else:
        m = mmap.mmap(-1, n, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        if mode == "mmap+THP":
            m.madvise(mmap.MADV_HUGEPAGE)
        b = np.frombuffer(m, dtype=np.int32)
    t0 = time.perf_counter(); torch.from_numpy(b).copy_(p); t1 = time.perf_counter()
    print(f"{mode}: fresh copy {n / (t1 - t0) / 1e9:.1f} GB/s", flush=True)
    t0 = time.perf_counter(); torch.from_numpy(b).copy_(p); t1 = time.perf_counter()
    print(f"{mode}: touched copy {n / (t1 - t0) / 1e9:.1f} GB/s", flush=True)
