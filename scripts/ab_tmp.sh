set -u
timeout 900 python -m pytest tests/test_gpu_pool.py -x -q > gpurun_out/r2q_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2q_pytest.log
mkdir -p gpurun_out/r2q
for env in "MF_UNPOOL_TMA=0" "MF_UNPOOL_TMA=1"; do
  env $env timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file "gpurun_out/r2q/launches_${env}.csv" python scripts/pool_step.py --warmup 1 > /dev/null 2>&1
  echo "== $env"; python scripts/launch_table.py "gpurun_out/r2q/launches_${env}.csv" --last 8
done
bash scripts/gpu_ab.sh r2q_ab MF_UNPOOL_TMA=0:cfg3 MF_UNPOOL_TMA=1:cfg3
