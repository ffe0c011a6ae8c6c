#!/bin/bash
# GPU parity run: pytest -m gpu (no -x: every failure listed) + smoke
# usage: tools/gpu_tests.sh TAG [pytest -k expr]
TAG=${1:-t}; K=${2:-}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $O/gpu.txt 2>&1
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -rs --durations=15 -k "$K" > $O/pytest_gpu.txt 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -q -rs --durations=15 > $O/pytest_gpu.txt 2>&1
fi
echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
echo done > $O/DONE
