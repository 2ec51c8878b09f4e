set -u
python -m pytest tests/test_gpu_chain.py -q -x 2>&1 | tail -2
bash scripts/gpu_ab.sh r2x MF_ZERO_COPY_IN=0:cfg2 MF_ZERO_COPY_IN=1:cfg2 MF_ZERO_COPY_IN=0:cfg2 MF_ZERO_COPY_IN=1:cfg2 MF_ZERO_COPY_IN=0:cfg5 MF_ZERO_COPY_IN=1:cfg5
