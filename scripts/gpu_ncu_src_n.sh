#!/bin/bash
# As gpu_ncu_src.sh, but capture the SKIP-th launch of the kernel (0-based) in the timed step.
#   gpurun -- 'bash scripts/gpu_ncu_src_n.sh <tag> <cfg> <kernel-regex> <skip>'
set -u
TAG=$1; CFG=$2; RX=$3; SKIP=$4
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s $SKIP -c 1 -f -o "$OUT/src" \
  python scripts/one_step.py --config $CFG --warmup 0 > "$OUT/ncu.log" 2>&1
echo "ncu rc=$?"
ncu -i "$OUT/src.ncu-rep" --page source --csv --print-source sass > "$OUT/src_sass.csv" 2>/dev/null
ncu -i "$OUT/src.ncu-rep" --page details > "$OUT/details.txt" 2>/dev/null
rm -f "$OUT/src.ncu-rep"
