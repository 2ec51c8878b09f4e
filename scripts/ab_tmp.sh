set -u
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_fullsize.py tests/test_gpu_fuzz.py -q -x 2>&1 | tail -2
bash scripts/gpu_ab.sh r3c MF_TWO_PASS_MIN=999999999:cfg5 -:cfg5 MF_TWO_PASS_MIN=999999999:cfg3 -:cfg3 MF_TWO_PASS_MIN=0:cfg3 MF_TWO_PASS_MIN=0:cfg2 -:cfg2 MF_TWO_PASS_MIN=0:cfg4 -:cfg4
