#!/bin/bash
# ncu --set full capture of selected kernels on one config (round 1 of its first level).
#   gpurun -- 'bash scripts/gpu_ncu.sh <tag> <cfg> <kernel-regex> [count]'
set -u
TAG=$1; CFG=$2; RX=$3; CNT=${4:-8}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { echo "build failed"; tail "$OUT/build.log"; }
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s 0 -c $CNT -f -o "$OUT/full_$CFG" \
  python scripts/one_step.py --config $CFG --warmup 1 > "$OUT/full_$CFG.log" 2>&1
echo "ncu rc=$?"; tail -3 "$OUT/full_$CFG.log"
