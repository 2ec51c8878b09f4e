#!/bin/bash
# A/B of a compile-time switch: bench runs with the default library, then with EXTRA nvcc flags.
#   gpurun -- 'bash scripts/gpu_ab_build.sh <tag> "<extra nvcc flags>" cfg2 cfg2 cfg5 ...'
set -u
TAG=$1; EXTRA=$2; shift 2
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
FLAGS="-O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall -gencode arch=compute_100a,code=sm_100a"
one() {
  local lab=$1 c=$2 i=$3
  case $c in cfg1|cfg2) S=100;; cfg3|cfg4) S=20;; *) S=5;; esac
  timeout 240 python bench.py --config $c --steps $S --warmup 3 --no-cpu-baseline > "$OUT/${lab}_$i.json" 2> "$OUT/${lab}_$i.err"
  echo "[$lab $c] rc=$? $(python -c "
import json;d=json.loads(open('$OUT/${lab}_$i.json').read().strip().splitlines()[-1])
print(round(d['ms_per_step'],4),'ms e2e',round(d['e2e']['ms_per_step'],3))" 2>&1)"
}
for lab in base var base2; do
  if [ $lab = var ]; then X="$EXTRA"; else X=""; fi
  rm -f paper_2103_15076_b200/libmfgpu.so
  make -C paper_2103_15076_b200/csrc NVFLAGS="$FLAGS $X" > "$OUT/build_$lab.log" 2>&1 || { echo "build $lab failed"; tail "$OUT/build_$lab.log"; }
  i=0
  for c in "$@"; do i=$((i+1)); one $lab $c $i; done
done
