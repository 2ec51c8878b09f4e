#!/bin/bash
# Source-level stall captures of several kernels of one config's step (first instance each).
#   gpurun -- 'bash scripts/gpu_ncu_multi.sh <tag> <cfg> <kernel-regex>...'
set -u
TAG=$1; CFG=$2; shift 2
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
i=0
for RX in "$@"; do
  i=$((i+1))
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s 0 -c 1 -f -o "$OUT/k$i" \
    python scripts/one_step.py --config $CFG --warmup 1 > "$OUT/k$i.log" 2>&1
  echo "ncu $RX rc=$?"
  mkdir -p "$OUT/k$i"
  ncu -i "$OUT/k$i.ncu-rep" --page source --csv --print-source sass > "$OUT/k$i/src_sass.csv" 2>/dev/null
  ncu -i "$OUT/k$i.ncu-rep" --page details > "$OUT/k$i/details.txt" 2>/dev/null
  ncu -i "$OUT/k$i.ncu-rep" --page raw --csv > "$OUT/k$i/raw.csv" 2>/dev/null
  rm -f "$OUT/k$i.ncu-rep"
done
