"""Key metrics of every launch in an ncu report (ncu -i REP --page details --csv) as a short text
summary: python tools/ncu_details.py REP.ncu-rep OUT.txt"""
import csv
import io
import subprocess
import sys

KEEP = ["Memory Throughput", "DRAM Throughput", "Duration", "Compute (SM) Throughput", "Issued Ipc Active",
        "L1/TEX Hit Rate", "L2 Hit Rate", "No Eligible", "Eligible Warps Per Scheduler", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Achieved Occupancy", "Block Limit Registers", "Waves Per SM"]


def main(rep, dst):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ii, ki, gi, mi, ui, vi = (hdr.index(k) for k in ("ID", "Kernel Name", "Grid Size", "Metric Name", "Metric Unit",
                                                     "Metric Value"))
    seen, lines, cur = set(), [], None
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        if r[ii] != cur:
            cur = r[ii]
            seen = set()
            lines.append(f"== launch {r[ii]} {r[ki][:60]} {r[gi]}")
        if r[mi] in KEEP and r[mi] not in seen:
            seen.add(r[mi])
            lines.append(f"   {r[mi]:<36} {r[ui]:>16} {r[vi]}")
    open(dst, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
