"""Digest an ncu report: python tools/ncu_digest.py rep.ncu-rep [kernel-regex]
Prints duration, IPC, pipes, stall reasons (per issue) and the SASS opcode mix."""
import csv, io, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
def page(p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))
r = page("raw")
h, u, v = r[0], r[1], r[2]
def g(n):
    return v[h.index(n)] if n in h else "?"
print("kernel:", g("Kernel Name"))
for n in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "launch__registers_per_thread", "launch__occupancy_limit_registers"]:
    print(f"  {n:55s} {g(n)} {u[h.index(n)] if n in h else ''}")
for i, n in enumerate(h):
    if n.startswith("sm__inst_executed_pipe_") and n.endswith(".avg.pct_of_peak_sustained_active"):
        try:
            if float(v[i]) > 2: print(f"  pipe {n[23:-33]:30s} {float(v[i]):6.1f} %")
        except ValueError: pass
st = []
for i, n in enumerate(h):
    if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
        st.append((float(v[i]), n[34:-23]))
print("  stalls/issue:", ", ".join(f"{k} {x:.2f}" for x, k in sorted(st, reverse=True) if x > 0.05))
s = page("source", ["--print-source", "sass"])
hh = s[1]; si = hh.index("Source"); ei = hh.index("Instructions Executed")
d = defaultdict(int); tot = 0
for x in s[2:]:
    try: n = int(x[ei].replace(",", ""))
    except (ValueError, IndexError): continue
    t = x[si].split()
    if not t: continue
    op = t[1] if t[0].startswith("@") else t[0]
    d[op] += n; tot += n
print("  opcode mix (share of warp instr):", ", ".join(f"{k} {c/tot*100:.1f}%" for k, c in sorted(d.items(), key=lambda t: -t[1])[:16]))
