"""Top warp-stall SASS lines of `ncu --page source --csv --print-source sass` exports.

    python scripts/stall_summary.py out.txt label=gpurun_out/src_edges/src_sass.csv ...

Each section lists the instructions holding the most stall samples (the sample lands on
the instruction that waits: the consumer of a pending load, atomic or barrier) plus the
kernel's duration / occupancy lines from the matching details.txt when present.
"""

import csv
import os
import sys


def main():
    out = [("# warp-stall samples by SASS instruction (ncu --set full --import-source on, "
            "source page); the waiting instruction carries the sample")]
    for arg in sys.argv[2:]:
        label, path = arg.split("=", 1)
        rows = list(csv.reader(open(path)))
        kname = rows[0][1] if len(rows[0]) > 1 else "?"
        rows = rows[2:]
        tot = sum(float(r[2] or 0) for r in rows) or 1.0
        out.append(f"\n== {label}: {kname.split('(')[0]}  ({int(tot)} samples)")
        det = os.path.join(os.path.dirname(path), "details.txt")
        if os.path.exists(det):
            for line in open(det):
                if any(k in line for k in ("Duration", "Achieved Occupancy", "Issue Slots Busy",
                                           "DRAM Throughput", "Registers Per Thread", "L2 Hit Rate")):
                    out.append("   " + " ".join(line.split()))
        recs = sorted(((float(r[2] or 0), r[0], r[1].strip()) for r in rows), reverse=True)[:12]
        for v, a, s in recs:
            out.append(f"  {100 * v / tot:5.1f}%  {hex(int(a, 16) & 0xffff):>7}  {s}")
    open(sys.argv[1], "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()
