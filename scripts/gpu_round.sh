#!/bin/bash
# One GPU-box pass: GPU tests, smoke, bench lines for every config (+ CPU baselines), the reference
# arm, ncu launch lists (cfg2, cfg5, the pooling half of cfg3) and `ncu --set full` captures of the
# hot kernels.
#   gpurun --timeout 3000 -- 'bash scripts/gpu_round.sh [tag] [parts]'
# parts: any of tests,bench,ncu (default all). Outputs land in gpurun_out/<tag>/.
set -u
TAG=${1:-run}
PARTS=${2:-tests,bench,ncu}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > "$OUT/gpu.txt" 2>&1
lscpu > "$OUT/lscpu.txt" 2>&1

if [[ $PARTS == *tests* ]]; then
  timeout 1500 python -m pytest tests -m gpu -q --timeout=900 > "$OUT/pytest_gpu.log" 2>&1; echo "pytest gpu rc=$?"
  tail -3 "$OUT/pytest_gpu.log"
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?"
  tail -1 "$OUT/smoke.log"
fi

if [[ $PARTS == *bench* ]]; then
  timeout 600 python bench.py > "$OUT/bench_default.json" 2> "$OUT/bench_default.err"; echo "bench default rc=$?"
  for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
    case $c in cfg1|cfg2) S=100;; cfg3|cfg4) S=20;; cfg5) S=5;; esac
    timeout 900 python bench.py --config $c --steps $S --warmup 3 > "$OUT/bench_$c.json" 2> "$OUT/bench_$c.err"
    echo "bench $c rc=$? $(python -c "import json,sys;d=json.loads(open('$OUT/bench_$c.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],4),'ms e2e',round(d['e2e']['ms_per_step'],3),'dom',d['roofline']['kernel'],round(d['roofline']['frac'] or 0,4))" 2>&1)"
  done
  timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"; echo "bench ref rc=$?"
fi

if [[ $PARTS == *ncu* ]]; then
  for c in cfg2 cfg5; do
    timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file "$OUT/launches_$c.csv" python scripts/one_step.py --config $c --warmup 3 > "$OUT/launches_$c.log" 2>&1
    echo "ncu launches $c rc=$?"
  done
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file "$OUT/launches_pool.csv" python scripts/pool_step.py --warmup 1 --fresh > "$OUT/launches_pool.log" 2>&1
  echo "ncu launches pool rc=$?"
  for c in cfg2 cfg5; do
    timeout 1500 ncu --set full --clock-control none --import-source on \
      -k regex:'k_suitor|k_vertex_t|k_edges|k_adj_rank|k_ld_pick|k_facet_remap|k_select|k_inc_scatter|k_facet_plane|k_scan_excl|k_init_inputs|k_contract|k_compose' \
      -s 0 -c 26 -f -o "$OUT/full_$c" \
      python scripts/one_step.py --config $c --warmup 1 > "$OUT/full_$c.log" 2>&1
    echo "ncu full $c rc=$?"
    ncu -i "$OUT/full_$c.ncu-rep" --page raw --csv > "$OUT/full_${c}_raw.csv" 2>/dev/null
    rm -f "$OUT/full_$c.ncu-rep"
  done
  timeout 900 ncu --set full --clock-control none -k regex:'k_pool|k_unpool|k_csr' -c 12 -f -o "$OUT/full_pool" \
    python scripts/pool_step.py --warmup 0 --fresh > "$OUT/full_pool.log" 2>&1
  echo "ncu full pool rc=$?"
  ncu -i "$OUT/full_pool.ncu-rep" --page raw --csv > "$OUT/full_pool_raw.csv" 2>/dev/null
  rm -f "$OUT/full_pool.ncu-rep"
fi
