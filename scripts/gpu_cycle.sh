#!/bin/bash
# Development cycle on one box: GPU tests, smoke, bench (cfg2 cfg3 cfg5 by default), ncu launch list of cfg2.
#   gpurun -- 'bash scripts/gpu_cycle.sh <tag> [cfgs...]'
set -u
TAG=${1:-cycle}; shift || true
CFGS=${@:-cfg2 cfg3 cfg5}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 1500 python -m pytest tests -m gpu -x -q --timeout=900 > "$OUT/pytest_gpu.log" 2>&1; echo "pytest gpu rc=$?"; tail -3 "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?"
for c in $CFGS; do
  case $c in cfg1|cfg2) S=100;; cfg3|cfg4) S=20;; *) S=5;; esac
  timeout 600 python bench.py --config $c --steps $S --warmup 3 --no-cpu-baseline > "$OUT/bench_$c.json" 2> "$OUT/bench_$c.err"
  echo "bench $c rc=$? $(python -c "
import json;d=json.loads(open('$OUT/bench_$c.json').read().strip().splitlines()[-1])
print(round(d['ms_per_step'],4),'ms e2e',round(d['e2e']['ms_per_step'],3),'launches',d['gpu_launches'],'dom',d['roofline']['kernel'],round(d['roofline']['frac'],4))
print('   ', ' '.join(f\"{k}={v['ms']:.4f}\" for k,v in list(d['kernels'].items())[:40]))" 2>&1)"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file "$OUT/launches_cfg2.csv" python scripts/one_step.py --config cfg2 --warmup 3 > "$OUT/launches_cfg2.log" 2>&1
echo "ncu cfg2 rc=$?"
python scripts/launch_table.py "$OUT/launches_cfg2.csv" --last 42
