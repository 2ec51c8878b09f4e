#!/bin/bash
set -u
OUT=gpurun_out/${1:-stress}; shift || true
mkdir -p "$OUT"
i=0
for spec in "$@"; do
  i=$((i+1)); envs=${spec%%:*}; c=${spec##*:}; [ "$envs" = "-" ] && envs=""
  env ${envs//,/ } timeout -k 10 -s INT 200 python scripts/stress.py --config $c --iters ${ITERS:-400} > "$OUT/s_$i.log" 2>&1
  echo "[$spec] rc=$? $(tail -1 $OUT/s_$i.log)"
  if ! grep -q STRESS-OK "$OUT/s_$i.log"; then tail -25 "$OUT/s_$i.log"; fi
done
