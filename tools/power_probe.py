"""Board power and SM clock while one kind of work runs back to back for
~3 s each (nvidia-smi sampled every 100 ms): the 16x16 NL kernel (tensor
cores + integer ALUs, no HBM traffic), an HBM copy (torch), the mask-major
spectrum kernel (compute + 4.3 GB of writes per call), and the 20x20 NL
(K3: both).  python tools/power_probe.py"""
import subprocess
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1912_03732_b200 as sw  # noqa: E402


def sample(fn, seconds=3.0):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=power.draw,clocks.sm,clocks_throttle_reasons.active",
                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    t0 = time.time()
    n = 0
    while time.time() - t0 < seconds:
        fn()
        n += 1
        torch.cuda.synchronize()
    p.terminate()
    out = p.communicate()[0].strip().splitlines()
    rows = [r.split(",") for r in out if r.strip()]
    rows = rows[len(rows) // 3:]  # steady state
    pw = sorted(float(r[0]) for r in rows)
    clk = sorted(float(r[1]) for r in rows)
    return n, pw[len(pw) // 2], clk[len(clk) // 2], sorted(set(r[2].strip() for r in rows))


s16 = sw.generate_sbox(16, 16, 0, bijective=True)
s20 = sw.generate_sbox(20, 20, 0, bijective=False)
x = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
y = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
out = torch.empty((16383, 65536), dtype=torch.int32, device="cuda")
sw.component_max_abs_device(s16)
cases = [("idle (sleep)", lambda: time.sleep(0.05)),
         ("16x16 NL (k_tc_hybrid<NL>)", lambda: sw.component_max_abs_device(s16)),
         ("HBM copy 4 GiB (torch)", lambda: y.copy_(x)),
         ("16x16 spectrum 4.3 GB (k_tc_hybrid<spec>)", lambda: sw.spectrum_device(s16, 1, 1 << 14, out=out)),
         ("20x20 NL, 65536 masks (K3)", lambda: sw.component_max_abs_device(s20, 1, 65537))]
for name, fn in cases:
    n, pw, clk, reasons = sample(fn)
    print(f"{name:45s} calls {n:5d}  median power {pw:6.0f} W  SM clock {clk:5.0f} MHz  reasons {reasons}", flush=True)
