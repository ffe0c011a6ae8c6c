#!/bin/bash
# quick GPU iteration: parity tests, SHVS + full bench lines, SHVS launch list
# usage: tools/gpu_iter.sh TAG [pytest -k expr]
TAG=${1:-it}; K=${2:-}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/$TAG; mkdir -p $O
if [ -n "$K" ]; then timeout 900 python -m pytest tests -m gpu -x -q -rs -k "$K" > $O/pytest_gpu.txt 2>&1; else timeout 900 python -m pytest tests -m gpu -x -q -rs > $O/pytest_gpu.txt 2>&1; fi
echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python bench.py --variant shvs --no-cpu-baseline --steps 300 > $O/bench_shvs.jsonl 2> $O/bench_shvs.err
timeout 300 python bench.py --no-cpu-baseline --steps 300 > $O/bench_full.jsonl 2> $O/bench_full.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file $O/launches_shvs.csv \
  python bench.py --variant shvs --steps 2 --warmup 3 --kernel-steps 2 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 300 python tools/phase_prof.py --variant shvs > $O/phase_shvs.txt 2>&1
echo done > $O/DONE
