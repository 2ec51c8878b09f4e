#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over the small fixtures,
# default path and every size-gated / A-B variant forced small.
#   gpurun --timeout 1800 -- 'bash scripts/gpu_sanitize.sh [tag]'
set -u
TAG=${1:-san}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool, label, env...
  local tool=$1 label=$2; shift 2
  env "$@" timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 50 \
    python scripts/sanitize_cases.py > "$OUT/${tool}_${label}.log" 2>&1
  echo "$tool $label rc=$? $(grep -E 'ERROR SUMMARY|SANITIZE-CASES-OK' "$OUT/${tool}_${label}.log" | tr '\n' ' ')"
}
for tool in memcheck racecheck synccheck; do
  run $tool default MF_SAN_N=20000
done
run memcheck variants_small MF_SAN_N=20000 MF_WIDE_MIN=0 MF_SCAN4_MIN=0 MF_BIG_SEL_MIN=0 MF_LD_MIN=1 MF_SUITOR=1
run racecheck variants_small MF_SAN_N=20000 MF_WIDE_MIN=0 MF_SCAN4_MIN=0 MF_BIG_SEL_MIN=0 MF_LD_MIN=1 MF_SUITOR=1
run memcheck suitor8_cluster MF_SAN_N=20000 MF_SUITOR=8 MF_SELECT_CL=1 MF_LD1_MIN=1
run racecheck suitor8_cluster MF_SAN_N=20000 MF_SUITOR=8 MF_SELECT_CL=1 MF_LD1_MIN=1
run memcheck nographs MF_SAN_N=20000 MF_GRAPHS=0
run memcheck pool_variants MF_SAN_N=20000 MF_UNPOOL_TMA=1 MF_CSR_COOP=0 MF_DEBUG=1
run racecheck pool_variants MF_SAN_N=20000 MF_UNPOOL_TMA=1 MF_CSR_COOP=0 MF_DEBUG=1
run synccheck pool_variants MF_SAN_N=20000 MF_UNPOOL_TMA=1
run memcheck fused_opt_in MF_SAN_N=20000 MF_VERTEX_SCAN=2 MF_EDGES_RANK=1 MF_VT16=1 MF_FUSE_PLANE=0
run racecheck fused_opt_in MF_SAN_N=20000 MF_VERTEX_SCAN=2 MF_EDGES_RANK=1 MF_VT16=1
run memcheck recompute_ticket MF_SAN_N=20000 MF_RECOMPUTE_MIN=0 MF_TWO_PASS_MIN=0 MF_SCAN_TICKET=1
run racecheck recompute_ticket MF_SAN_N=20000 MF_RECOMPUTE_MIN=0 MF_TWO_PASS_MIN=0 MF_SCAN_TICKET=1
run initcheck default MF_SAN_N=20000 MF_GRAPHS=0
