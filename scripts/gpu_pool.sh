#!/bin/bash
# Pool / unpool pass: parity tests, cfg3 bench, ncu launch list + full capture of the pool kernels.
set -u
TAG=${1:-pool}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_gpu_pool.py tests/test_gpu_golden.py "tests/test_gpu_fullsize.py::test_full_size_matches_oracle[cfg3]" "tests/test_gpu_fullsize.py::test_full_size_matches_reference[cfg3]" -x -q > "$OUT/pytest.log" 2>&1; echo "pytest rc=$?"; tail -2 "$OUT/pytest.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?"
for c in cfg3 cfg2; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > "$OUT/bench_$c.json" 2> "$OUT/bench_$c.err"
  echo "bench $c rc=$? $(python -c "
import json;d=json.loads(open('$OUT/bench_$c.json').read().strip().splitlines()[-1])
print(round(d['ms_per_step'],4),'ms e2e',round(d['e2e']['ms_per_step'],3),'dom',d['roofline']['kernel'],round(d['roofline']['frac'],4))
print('   ', ' '.join(f\"{k}={v['ms']:.4f}\" for k,v in list(d['kernels'].items())[:40]))" 2>&1)"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file "$OUT/launches_pool.csv" python scripts/pool_step.py --warmup 1 --fresh > "$OUT/launches_pool.log" 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_pool|k_unpool|k_count_keys|k_csr|k_seg_sort' \
  -c 16 -f -o "$OUT/full_pool" python scripts/pool_step.py --warmup 0 --fresh > "$OUT/full_pool.log" 2>&1
echo "ncu full rc=$?"
ncu -i "$OUT/full_pool.ncu-rep" --page raw --csv > "$OUT/full_pool_raw.csv" 2>/dev/null
ncu -i "$OUT/full_pool.ncu-rep" --page details > "$OUT/full_pool_details.txt" 2>/dev/null
if [ -f "$OUT/full_pool.ncu-rep" ] && [ $(stat -c %s "$OUT/full_pool.ncu-rep") -gt 20000000 ]; then rm -f "$OUT/full_pool.ncu-rep"; fi
