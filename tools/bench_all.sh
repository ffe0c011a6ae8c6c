#!/bin/bash
# run the bench on every config (one GPU); one JSON line each into gpurun_out/$TAG/bench_<cfg>.jsonl
TAG=${1:-all}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/$TAG; mkdir -p $O
run() { local name=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$name.jsonl 2> $O/bench_$name.err; }
run c2 --steps 1000 --warmup 10 --cpu-seconds 10
run c2_shvs --config c2 --variant shvs --steps 500 --warmup 5 --no-cpu-baseline
run c1 --config c1 --steps 1000 --warmup 10 --no-cpu-baseline
run c3 --config c3 --steps 300 --warmup 5 --no-cpu-baseline
run c5 --config c5 --steps 50 --warmup 3 --no-cpu-baseline
run c5_full --config c5 --variant full --steps 30 --warmup 3 --no-cpu-baseline --no-shvs
run c4 --config c4 --steps 50 --warmup 3 --no-cpu-baseline
run c2long --config c2long --steps 100 --warmup 5 --no-cpu-baseline
run ref --impl reference --steps 5 --warmup 3
