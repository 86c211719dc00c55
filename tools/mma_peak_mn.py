"""tcgen05.mma.kind::i8 128x256x32 chain rate with B K-major (SBW_PEAK_MN=0) vs
MN-major SWIZZLE_128B (SBW_PEAK_MN=1), one subprocess each."""
import os
import subprocess
import sys

code = r'''
import ctypes as c, sys, torch
sys.path.insert(0, ".")
from paper_1912_03732_b200 import device
lib = device.load_library()
d = torch.device("cuda:0"); torch.zeros(1, device=d)
best = 0
for _ in range(3):
    ops, ms = c.c_double(), c.c_double()
    rc = lib.sbw_int8_mma_peak(c.byref(ops), c.byref(ms), device.stream_handle(d))
    best = max(best, ops.value)
print(f"{best/1e15:.3f} POP/s")
'''
for mn in ("0", "1"):
    p = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, SBW_PEAK_MN=mn), capture_output=True, text=True)
    print(f"SBW_PEAK_MN={mn}: {p.stdout.strip() or p.stderr.strip()[-500:]}", flush=True)
