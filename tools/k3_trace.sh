# timeline of the batched multi-pass path (SBW_K3_TRACE) + raw HBM write/read rates
SBW_K3_TRACE=1 timeout 120 python tools/k3_probe.py 20x20 32768
SBW_K3_TRACE=1 timeout 120 python tools/k3_probe.py 24x16 1024
python - <<'PY'
import torch
x = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
for name, f in [("write (fill_)", lambda: x.fill_(1)), ("read (sum int64 via view)", lambda: x.view(torch.int64).sum()),
                ("copy", lambda: x[: 2 << 30].copy_(x[2 << 30 :]))]:
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    nbytes = 4 << 30
    print(name, f"{best:.3f} ms", f"{nbytes / best / 1e9:.0f} GB/s")
PY
