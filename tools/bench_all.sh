#!/bin/bash
# run the bench on several configs (one GPU); one JSON line each into gpurun_out/bench_$TAG.jsonl
TAG=$1
cd "${GRAFT_REPO_ROOT:-/root/repo}"
: > gpurun_out/bench_$TAG.jsonl
run() { timeout 600 python bench.py "$@" 2> gpurun_out/bench_err_$TAG.txt | tail -1 >> gpurun_out/bench_$TAG.jsonl; }
run --steps 1000 --warmup 10 --cpu-seconds 10
run --config c2 --variant shvs --steps 500 --warmup 5 --no-cpu-baseline
run --config c1 --steps 1000 --warmup 10 --no-cpu-baseline
run --config c5 --steps 50 --warmup 3 --no-cpu-baseline
run --config c4 --steps 50 --warmup 3 --no-cpu-baseline
