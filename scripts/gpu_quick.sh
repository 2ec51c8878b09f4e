#!/bin/bash
# Quick GPU pass: build, GPU tests, bench on the given configs (default cfg2 cfg5).
#   gpurun -- 'bash scripts/gpu_quick.sh <tag> [cfgs...]'
set -u
TAG=${1:-quick}; shift || true
CFGS=${@:-cfg2 cfg5}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || { echo "build failed"; tail "$OUT/build.log"; }
timeout 900 python -m pytest tests -m gpu -x -q --timeout=120 > "$OUT/pytest_gpu.log" 2>&1; echo "pytest gpu rc=$?"; tail -3 "$OUT/pytest_gpu.log"
for c in $CFGS; do
  case $c in cfg1|cfg2) S=100;; cfg3|cfg4) S=20;; *) S=5;; esac
  timeout 600 python bench.py --config $c --steps $S --warmup 3 --no-cpu-baseline > "$OUT/bench_$c.json" 2> "$OUT/bench_$c.err"
  echo "bench $c rc=$? $(python -c "
import json;d=json.loads(open('$OUT/bench_$c.json').read().strip().splitlines()[-1])
print(round(d['ms_per_step'],4),'ms e2e',round(d['e2e']['ms_per_step'],3),'dom',d['roofline']['kernel'],round(d['roofline']['frac'],4))
print('   ', ' '.join(f\"{k}={v['ms']:.3f}\" for k,v in list(d['kernels'].items())[:12]))" 2>&1)"
done
