"""Mean DRAM bytes per MG-sweep launch (k_wave<1, 0>) from an ncu --metrics
dram__bytes_read.sum,dram__bytes_write.sum --csv launch list -> profiles/traffic.json."""
import collections
import csv
import json
import sys


def main(src, dst, key, note):
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    ii = hdr.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        if r[mi].startswith("dram__bytes"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        per[r[ii]][r[mi]] = v
        names[r[ii]] = r[ki]
    sweeps = [k for k in per if names[k].startswith("void k_wave<1, 0>") or names[k].startswith("void k_wave<0, 0>")]
    tot = [per[k]["dram__bytes_read.sum"] + per[k]["dram__bytes_write.sum"] for k in sweeps]
    out = {key: sum(tot) / len(tot), "launches": len(tot), "note": note}
    json.dump(out, open(dst, "w"), indent=1)
    print(out)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], " ".join(sys.argv[4:]))
