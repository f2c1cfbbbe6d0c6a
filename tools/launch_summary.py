"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel + launch shape."""
import collections
import csv
import sys


def main(src, dst, note=""):
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    gi, bi = hdr.index("Grid Size"), hdr.index("Block Size")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        k = r[ki].split("(")[0] + " grid" + r[gi] + " block" + r[bi]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    tot = sum(a[1] for a in agg.values())
    with open(dst, "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)\n")
        if note:
            f.write(f"# {note}\n")
        f.write(f"# total kernel time {tot / 1e6:.3f} ms over {len(rows) - 1} launches\n")
        for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{a[1] / 1e6:9.3f} ms {100 * a[1] / tot:5.1f}%  n={a[0]:5d}  avg={a[1] / a[0] / 1e3:9.1f} us  {k}\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], " ".join(sys.argv[3:]))
