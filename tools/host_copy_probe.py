import time, torch, numpy as np
dev = torch.device("cuda", 0)
x = torch.empty(1 << 29, dtype=torch.int32, device=dev)  # 2 GiB
x.fill_(7)
torch.cuda.synchronize()
for gb in (2, 16):
    t0 = time.perf_counter(); p = torch.empty((gb << 28,), dtype=torch.int32, pin_memory=True); t1 = time.perf_counter()
    print(f"pinned alloc {gb} GiB: {t1-t0:.3f} s")
    t0 = time.perf_counter(); p[: 1 << 29].copy_(x); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"D2H 2 GiB into pinned: {(2<<30)/(t1-t0)/1e9:.1f} GB/s")
    t0 = time.perf_counter(); p[: 1 << 29].copy_(x); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"D2H 2 GiB into pinned (2nd): {(2<<30)/(t1-t0)/1e9:.1f} GB/s")
    del p
a = np.empty(1 << 29, dtype=np.int32)
t0 = time.perf_counter(); a[:] = 1; t1 = time.perf_counter(); print(f"numpy first-touch fill 2 GiB: {(2<<30)/(t1-t0)/1e9:.1f} GB/s")
p = torch.empty((1 << 29,), dtype=torch.int32, pin_memory=True); p.fill_(3)
b = np.empty(1 << 29, dtype=np.int32)
t0 = time.perf_counter(); torch.from_numpy(b).copy_(p); t1 = time.perf_counter(); print(f"torch copy pinned->fresh numpy 2 GiB: {(2<<30)/(t1-t0)/1e9:.1f} GB/s, threads {torch.get_num_threads()}")
t0 = time.perf_counter(); torch.from_numpy(b).copy_(p); t1 = time.perf_counter(); print(f"torch copy pinned->touched numpy 2 GiB: {(2<<30)/(t1-t0)/1e9:.1f} GB/s")
t0 = time.perf_counter(); r = torch.cuda.cudart().cudaHostRegister(b.ctypes.data, b.nbytes, 0); t1 = time.perf_counter(); print(f"cudaHostRegister 2 GiB: {t1-t0:.3f} s rc={r}")
bt = torch.from_numpy(b)
t0 = time.perf_counter(); bt.copy_(x, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter(); print(f"D2H into registered numpy: {(2<<30)/(t1-t0)/1e9:.1f} GB/s")
import sys; sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw
s = sw.generate_sbox(16, 16, 0, bijective=True)
for _ in range(2):
    t0 = time.perf_counter(); out, mx = sw.spectrum_to_host(s, 1, 1 << 14); t1 = time.perf_counter()
    print(f"spectrum_to_host 16383 rows (4.3 GB): {t1-t0:.3f} s = {4.29/(t1-t0):.1f} GB/s")
    del out
