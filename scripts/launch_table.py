"""Print an ncu launch list (--metrics gpu__time_duration.sum[,dram__bytes_*]) as a table.

    python scripts/launch_table.py launches.csv [--last N] [--from-kernel NAME]"""
import csv
import sys
from collections import OrderedDict

path = sys.argv[1]
last = int(sys.argv[sys.argv.index("--last") + 1]) if "--last" in sys.argv else 0
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
k = OrderedDict()
for d in data:
    it = k.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0][:48], "grid": d["Grid Size"]})
    it[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
items = list(k.values())[-last:] if last else list(k.values())
tot = 0.0
for it in items:
    t = it.get("gpu__time_duration.sum", 0) / 1000
    rb = it.get("dram__bytes_read.sum", 0) / 1e6
    wb = it.get("dram__bytes_write.sum", 0) / 1e6
    tot += t
    print("%-48s %8.2f us  R %8.2f MB  W %8.2f MB  %6.0f GB/s  %s" % (it["name"], t, rb, wb,
                                                                   (rb + wb) / t * 1e3 if t else 0, it["grid"]))
print("total %.2f us over %d launches" % (tot, len(items)))
