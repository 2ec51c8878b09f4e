#!/bin/bash
# Cheap per-launch DRAM / duration metrics for selected kernels on one config.
#   gpurun -- 'bash scripts/gpu_ncu_metrics.sh <tag> <cfg> <kernel-regex> [count]'
set -u
TAG=$1; CFG=$2; RX=$3; CNT=${4:-8}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { echo "build failed"; tail "$OUT/build.log"; }
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read.sum \
  --clock-control none -k regex:"$RX" -s 0 -c $CNT --csv python scripts/one_step.py --config $CFG --warmup 1 > "$OUT/m_$CFG.csv" 2> "$OUT/m_$CFG.err"
echo "ncu rc=$?"
python - "$OUT/m_$CFG.csv" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; ki, mi, ui, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
by = {}
for r in rows[1:]:
    by.setdefault((r[ii], r[ki].split("(")[0]), {})[r[mi]] = (r[vi], r[ui])
for (i, k), m in by.items():
    print(i, k, " ".join(f"{n.split('__')[1][:28]}={v}{u}" for n, (v, u) in sorted(m.items())))
PY
