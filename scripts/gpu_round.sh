#!/bin/bash
# One GPU-box pass: GPU tests, smoke, bench lines for every config, the reference
# arm, an ncu launch list and one `ncu --set full` capture of the hot kernels.
#   gpurun --timeout 2400 -- 'bash scripts/gpu_round.sh [tag] [parts]'
# parts: any of tests,bench,ncu (default all). Outputs land in gpurun_out/<tag>/.
set -u
TAG=${1:-run}
PARTS=${2:-tests,bench,ncu}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > "$OUT/gpu.txt" 2>&1
python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1 || echo "build failed"

if [[ $PARTS == *tests* ]]; then
  timeout 1200 python -m pytest tests -m gpu -x -q --timeout=120 > "$OUT/pytest_gpu.log" 2>&1; echo "pytest gpu rc=$?"
  tail -3 "$OUT/pytest_gpu.log"
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?"
  tail -1 "$OUT/smoke.log"
fi

if [[ $PARTS == *bench* ]]; then
  timeout 300 python bench.py > "$OUT/bench_default.json" 2> "$OUT/bench_default.err"; echo "bench default rc=$?"
  for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
    case $c in cfg1|cfg2) S=100;; cfg3|cfg4) S=20;; cfg5) S=5;; esac
    timeout 600 python bench.py --config $c --steps $S --warmup 3 > "$OUT/bench_$c.json" 2> "$OUT/bench_$c.err"
    echo "bench $c rc=$? $(python -c "import json,sys;d=json.loads(open('$OUT/bench_$c.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],'ms e2e',d['e2e']['ms_per_step'],'dom',d['roofline']['kernel'],round(d['roofline']['frac'],4))" 2>&1)"
  done
  timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"; echo "bench ref rc=$?"
fi

if [[ $PARTS == *ncu* ]]; then
  for c in cfg2 cfg5; do
    W=3
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file "$OUT/launches_$c.csv" python scripts/one_step.py --config $c --warmup $W > "$OUT/launches_$c.log" 2>&1
    echo "ncu launches $c rc=$?"
  done
  for c in cfg2 cfg5; do
    timeout 1500 ncu --set full --clock-control none --import-source on \
      -k regex:'k_suitor|k_vertex_t|k_edges|k_adj_rank|k_ld_pick|k_facet_remap|k_select|k_inc_scatter|k_facet_plane|k_scan_excl' \
      -s 0 -c 24 -f -o "$OUT/full_$c" \
      python scripts/one_step.py --config $c --warmup 1 > "$OUT/full_$c.log" 2>&1
    echo "ncu full $c rc=$?"
    # keep the merge-back small: CSV / text exports, the report itself only when small
    ncu -i "$OUT/full_$c.ncu-rep" --page raw --csv > "$OUT/full_${c}_raw.csv" 2>/dev/null
    ncu -i "$OUT/full_$c.ncu-rep" --page details > "$OUT/full_${c}_details.txt" 2>/dev/null
    if [ -f "$OUT/full_$c.ncu-rep" ] && [ $(stat -c %s "$OUT/full_$c.ncu-rep") -gt 20000000 ]; then rm -f "$OUT/full_$c.ncu-rep"; fi
  done
fi
