"""Print an ncu --csv launch list compactly: id, kernel, duration (us), DRAM MB read/written."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
acc = {}
order = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k = (int(d["ID"]), d["Kernel Name"])
        if k not in acc:
            acc[k] = {}
            order.append(k)
        acc[k][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
for k in order:
    m = acc[k]
    print(f"{k[0]:4d} {k[1][:58]:58s} {m.get('gpu__time_duration.sum', 0) / 1e3:9.1f} us "
          f"rd {m.get('dram__bytes_read.sum', 0) / 1e6:8.1f} MB wr {m.get('dram__bytes_write.sum', 0) / 1e6:8.1f} MB")
