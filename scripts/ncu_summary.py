"""Summarise `ncu --set full` captures into profiles/.

    python scripts/ncu_summary.py <tag> cfg2=gpurun_out/r/full_cfg2.ncu-rep cfg5=...

Writes profiles/<tag>_ncu_full_summary.txt (per launch: duration, DRAM bytes,
DRAM / L2 / occupancy figures) and merges per-kernel DRAM traffic per launch
(dram__bytes_read.sum + dram__bytes_write.sum, averaged over the captured
launches of that kernel) into profiles/ncu_traffic.json, which bench.py reads
for `roofline.traffic`.
"""

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COLS = {
    "dur_us": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_hit": "lts__t_sector_hit_rate.pct",
    "occ": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}
SCALE = {"ms": 1e3, "us": 1.0, "ns": 1e-3, "usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def kname(raw: str) -> str:
    s = raw.split("(")[0]
    return s[5:] if s.startswith("void ") else s


def read(rep: str):
    if rep.endswith(".csv"):  # a `--page raw --csv` export made next to the capture
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        rec = {"kernel": kname(r[head.index("Kernel Name")])}
        for key, col in COLS.items():
            if col not in head:
                rec[key] = None
                continue
            i = head.index(col)
            try:
                val = float(r[i].replace(",", ""))
            except ValueError:
                rec[key] = None
                continue
            u = units[i]
            if key == "dur_us":
                val *= SCALE.get(u, 1.0)
            elif key in ("dram_rd", "dram_wr"):
                val *= SCALE.get(u, 1.0)
            rec[key] = val
        recs.append(rec)
    return recs


def main():
    tag = sys.argv[1]
    lines = [f"# ncu --set full --clock-control none summaries ({tag}); per launch, cold-cache replay",
             "# columns: kernel | duration us | DRAM read MB | DRAM write MB | achieved GB/s | DRAM % peak | L2 hit % | "
             "warps active % | regs | grid x block"]
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(tp)) if os.path.exists(tp) else {}
    for arg in sys.argv[2:]:
        cfg, rep = arg.split("=", 1)
        recs = read(rep)
        lines.append(f"== {cfg}: {os.path.basename(rep)}")
        agg = {}
        for r in recs:
            rd, wr, d = r["dram_rd"] or 0.0, r["dram_wr"] or 0.0, r["dur_us"] or 0.0
            gbs = (rd + wr) / (d * 1e3) if d else 0.0
            lines.append(f"{r['kernel']:28s} {d:9.1f} {rd / 1e6:9.1f} {wr / 1e6:9.1f} {gbs:8.0f} "
                         f"{(r['dram_pct'] or 0):6.1f} {(r['l2_hit'] or 0):6.1f} {(r['occ'] or 0):6.1f} "
                         f"{int(r['regs'] or 0):4d} {int(r['grid'] or 0)}x{int(r['block'] or 0)}")
            a = agg.setdefault(r["kernel"], [0.0, 0])
            a[0] += rd + wr
            a[1] += 1
        traffic.setdefault(cfg, {}).update({k: v[0] / v[1] for k, v in agg.items()})
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full_summary.txt"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    with open(tp, "w") as fh:
        json.dump(traffic, fh, indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
