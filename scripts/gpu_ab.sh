#!/bin/bash
# A/B bench runs: each argument is "ENV=VAL,ENV2=VAL2:cfg" (use "-" for no env).
#   gpurun -- 'bash scripts/gpu_ab.sh <tag> -:cfg2 MF_SUITOR=8:cfg2'
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { echo "build failed"; tail "$OUT/build.log"; }
if [ "${AB_TESTS:-0}" = "1" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q --timeout=120 > "$OUT/pytest_gpu.log" 2>&1; echo "pytest gpu rc=$?"; tail -2 "$OUT/pytest_gpu.log"
fi
i=0
for spec in "$@"; do
  envs=${spec%%:*}; c=${spec##*:}
  case $c in cfg1|cfg2) S=100;; cfg3|cfg4) S=20;; *) S=5;; esac
  i=$((i+1))
  if [ "$envs" = "-" ]; then envs=""; fi
  env ${envs//,/ } timeout 240 python bench.py --config $c --steps $S --warmup 3 --no-cpu-baseline > "$OUT/ab_$i.json" 2> "$OUT/ab_$i.err"
  echo "[$spec] rc=$? $(python -c "
import json;d=json.loads(open('$OUT/ab_$i.json').read().strip().splitlines()[-1])
print(round(d['ms_per_step'],4),'ms e2e',round(d['e2e']['ms_per_step'],3))
print('   ', ' '.join(f\"{k}={v['ms']:.3f}\" for k,v in list(d['kernels'].items())[:14]))" 2>&1)"
done
