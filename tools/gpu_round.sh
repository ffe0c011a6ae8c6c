#!/bin/bash
# one GPU round-trip: parity tests, split sweep, ncu of the top kernel
# usage: tools/gpu_round.sh TAG [extra bench args]
TAG=$1; shift
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 python -m pytest tests -m gpu -x -q -rs > gpurun_out/pytest_gpu_$TAG.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.txt
for s in 0 1 2 4; do timeout 120 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --split $s "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($s, round(d['value']), round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],4))" >> gpurun_out/split_$TAG.txt 2>&1; done
ncu --set full --clock-control none --import-source on -k regex:"topk_sample|stream_sample" -s 1 -c 1 -o gpurun_out/prof_$TAG python tools/prof_step.py --steps 3 > gpurun_out/ncu_$TAG.txt 2>&1
python tools/stats_c2.py > gpurun_out/stats_$TAG.txt 2>&1
