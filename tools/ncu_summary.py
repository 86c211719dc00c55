"""Summarise an ncu report (run here, no GPU): key throughput metrics, DRAM
traffic, pipe utilisation, stall reasons and the dynamic SASS opcode mix.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--elements N] [--json out.json] > summary.md
"""
import argparse
import collections
import csv
import io
import json
import subprocess


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--elements", type=float, default=0, help="algorithmic elements per launch")
    ap.add_argument("--json", default="")
    a = ap.parse_args()

    raw = ncu_csv(a.rep, "--page", "raw")
    hdr, vals = raw[0], raw[2]
    d = dict(zip(hdr, vals))
    name = d.get("Kernel Name", "?")

    def f(key):
        try:
            return float(d[key].replace(",", ""))
        except (KeyError, ValueError):
            return float("nan")

    dur_ns = f("gpu__time_duration.sum")
    dram = f("dram__bytes_read.sum") + f("dram__bytes_write.sum")
    # dram__bytes_* are reported in the unit row; normalise to bytes
    units = dict(zip(hdr, raw[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    dram = (f("dram__bytes_read.sum") * scale.get(units.get("dram__bytes_read.sum", "byte"), 1)
            + f("dram__bytes_write.sum") * scale.get(units.get("dram__bytes_write.sum", "byte"), 1))
    dur_scale = {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(
        units.get("gpu__time_duration.sum", "nsecond"), 1)
    dur_ns *= dur_scale

    print(f"# ncu summary: `{name}`\n")
    print(f"report: `{a.rep}`\n")
    rows = [
        ("duration", f"{dur_ns / 1e3:.1f} us"),
        ("SM frequency", f"{f('smsp__cycles_elapsed.avg.per_second'):.2f} "
                         f"{units.get('smsp__cycles_elapsed.avg.per_second', '')}"),
        ("DRAM bytes (read+write)", f"{dram:,.0f}"),
        ("issue slots busy", f"{f('sm__instruction_throughput.avg.pct_of_peak_sustained_active'):.1f} %"),
        ("executed IPC (active)", f"{f('sm__inst_executed.avg.per_cycle_active'):.2f}"),
        ("ALU pipe", f"{f('sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active'):.1f} %"),
        ("FMA pipe", f"{f('sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'):.1f} %"),
        ("LSU pipe", f"{f('sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active'):.1f} %"),
        ("XU pipe", f"{f('sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active'):.1f} %"),
        ("achieved occupancy", f"{f('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} %"),
        ("registers/thread", f"{f('launch__registers_per_thread'):.0f}"),
        ("smem bank conflicts (ld+st)",
         f"{f('l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum') + f('l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum'):,.0f}"),
    ]
    print("| metric | value |\n|---|---|")
    for k, v in rows:
        print(f"| {k} | {v} |")

    stalls = {h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""):
              f(h) for h in hdr if h.startswith("smsp__average_warps_issue_stalled_")
              and h.endswith("per_issue_active.ratio")}
    print("\n## stall reasons (warps per issued instruction)\n\n| reason | ratio |\n|---|---|")
    for k, v in sorted(stalls.items(), key=lambda kv: -kv[1]):
        if v >= 0.02:
            print(f"| {k} | {v:.3f} |")

    src = ncu_csv(a.rep, "--page", "source", "--print-source", "sass")
    total = 0
    mix = collections.Counter()
    if len(src) > 2:
        h = src[1]
        ie, sc = h.index("Instructions Executed"), h.index("Source")
        for r in src[2:]:
            toks = r[sc].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") else toks[0]
            n = int(r[ie] or 0)
            mix[op] += n
            total += n
    print(f"\n## dynamic SASS mix\n\nwarp instructions: {total:,}")
    if a.elements:
        print(f"; thread-instructions per element: {total * 32 / a.elements:.2f}")
    print("\n| opcode | warp instr | per element |\n|---|---|---|")
    for op, n in mix.most_common(18):
        per = f"{n * 32 / a.elements:.3f}" if a.elements else ""
        print(f"| {op} | {n:,} | {per} |")

    if a.json:
        with open(a.json, "w") as fh:
            json.dump({"kernel": name, "duration_us": dur_ns / 1e3,
                       "dram_bytes_per_launch": dram, "warp_instructions": total,
                       "thread_instr_per_element": total * 32 / a.elements if a.elements else None,
                       "source": a.rep}, fh, indent=1)


if __name__ == "__main__":
    main()
