"""Top stalled SASS instructions of an ncu report (source page): python tools/ncu_top_stalls.py X.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try: return float(r[ix[k]])
    except Exception: return 0.0
tot = sum(f(r, '# Samples') for r in data)
print("total samples", int(tot))
keys = ['stall_long_sb', 'stall_short_sb', 'stall_mio', 'stall_math', 'stall_wait', 'stall_sleep', 'stall_barrier', 'stall_membar']
for r in sorted(data, key=lambda r: -f(r, '# Samples'))[:n]:
    print(r[ix['Address']][-5:], f"{100*f(r,'# Samples')/tot:5.1f}%", ' '.join(f"{k[6:]}={int(f(r,k))}" for k in keys if f(r, k) > 0), '|', r[ix['Source']][:80])
