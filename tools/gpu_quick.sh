#!/bin/bash
# quick GPU iteration: full gpu pytest + smoke + C2 bench at 20 and 1000 steps (+ SHVS)
TAG=${1:-q}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/$TAG; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -rs -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_c2_20.json 2> $O/bench.err
timeout 600 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline > $O/bench_c2_1000.json 2>> $O/bench.err
echo done > $O/DONE
