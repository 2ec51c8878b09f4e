bash scripts/gpu_cycle.sh r2o cfg2 cfg3 cfg5
bash scripts/gpu_ab.sh r2o_ab MF_VT16=0:cfg2 -:cfg2 MF_VT16=0:cfg2 -:cfg2
