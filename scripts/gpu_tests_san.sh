#!/bin/bash
# GPU test suite + sanitizer pass in one box session.
set -u
TAG=${1:-r2a}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > "$OUT/gpu.txt" 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout=900 -x --durations=15 > "$OUT/pytest_gpu.log" 2>&1; echo "pytest gpu rc=$?"
tail -25 "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?"
bash scripts/gpu_sanitize.sh $TAG/san
