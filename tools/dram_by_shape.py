"""Per launch shape: mean duration, DRAM bytes and GB/s from an ncu --metrics
dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, gi, bi, mi, vi, ui, ii = (h.index(k) for k in ("Kernel Name", "Grid Size", "Block Size", "Metric Name",
                                                   "Metric Value", "Metric Unit", "ID"))
per, shape = collections.defaultdict(dict), {}
for r in rows[1:]:
    v = float(r[vi].replace(",", ""))
    if r[mi].startswith("dram"):
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[ui], 1)
    if r[mi] == "gpu__time_duration.sum":
        v *= {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3}.get(r[ui], 1)
    per[r[ii]][r[mi]] = v
    shape[r[ii]] = (r[ki][:20], r[gi], r[bi])
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for k, d in per.items():
    a = agg[shape[k]]
    a[0] += 1
    a[1] += d["gpu__time_duration.sum"]
    a[2] += d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
for s, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(*s, n, f"{t / n / 1e3:.1f} us", f"{b / n / 1e6:.1f} MB", f"{b / t:.0f} GB/s")
