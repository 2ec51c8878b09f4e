#!/bin/bash
set -u
TAG=${1:-poolq}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_gpu_pool.py tests/test_gpu_golden.py -x -q > "$OUT/pytest.log" 2>&1; echo "pytest rc=$?"; tail -2 "$OUT/pytest.log"
for env in "MF_CSR_COOP=1" "MF_CSR_COOP=0"; do
  env $env timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file "$OUT/launches_pool_${env}.csv" python scripts/pool_step.py --warmup 1 --fresh > "$OUT/launches_pool_${env}.log" 2>&1
  echo "ncu $env rc=$?"
  python scripts/launch_table.py "$OUT/launches_pool_${env}.csv" --last 24 | grep -v "k_pool_vec\|k_unpool"
done
