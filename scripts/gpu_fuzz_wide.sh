#!/bin/bash
# Wider fuzz sweep: extra seeds on the defaults, and the base seeds under forced size gates.
#   gpurun -- 'bash scripts/gpu_fuzz_wide.sh <tag> [a:b]'
set -u
TAG=$1; SEEDS=${2:-120:620}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { echo "build failed"; tail "$OUT/build.log"; }
run() {
  local name=$1; shift
  env "$@" timeout 1500 python -m pytest tests/test_gpu_fuzz.py -q -n 6 -p no:cacheprovider > "$OUT/fuzz_$name.log" 2>&1
  echo "[$name] rc=$? $(tail -1 "$OUT/fuzz_$name.log")"
}
run defaults MF_FUZZ_SEEDS=$SEEDS
run gates MF_FUZZ_SEEDS=${VSEEDS:-0:120} MF_WIDE_MIN=0 MF_SCAN4_MIN=0 MF_BIG_SEL_MIN=0 MF_LD_MIN=1 MF_LD1_MIN=1
run suitor8_nographs MF_FUZZ_SEEDS=${VSEEDS:-0:120} MF_SUITOR=8 MF_GRAPHS=0
run recompute_vt16 MF_FUZZ_SEEDS=${VSEEDS:-0:120} MF_RECOMPUTE_MIN=0 MF_VT16=1 MF_TWO_PASS_MIN=0
