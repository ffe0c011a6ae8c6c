#!/bin/bash
# C5 full-path analysis: per-row-kind K1 timeline, phase clocks, launch list
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${1:-c5an}; mkdir -p $O
DP_LIB=paper_2512_00719_b200/_lib/variants/timeline.so timeout 600 python tools/micro/timeline.py --config c5 > $O/timeline_c5.txt 2>&1
timeout 600 python tools/phase_prof.py --config c5 --variant full > $O/phase_c5_full.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_c5_full.csv python tools/prof_step.py --config c5 --variant full --steps 3 > $O/prof.log 2>&1
timeout 600 python bench.py --config c5 --variant full --steps 30 --warmup 3 --no-cpu-baseline --no-shvs > $O/bench_c5_full.jsonl 2> $O/bench.err
echo done > $O/DONE
