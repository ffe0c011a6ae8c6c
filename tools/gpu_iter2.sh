#!/bin/bash
# one iteration: GPU parity, C5 per-kind timeline, bench lines of the full path (c2, c4, c5, c1)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${1:-it}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
[ -f paper_2512_00719_b200/_lib/variants/timeline.so ] && DP_LIB=paper_2512_00719_b200/_lib/variants/timeline.so timeout 600 python tools/micro/timeline.py --config c5 > $O/timeline_c5.txt 2>&1
b() { local n=$1; shift; timeout 600 python bench.py "$@" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d.get('shvs') or {}; print('$n', round(d['ms_per_step']*1000,1), 'us frac', round(d['roofline']['frac'],3), 'shvs', s.get('hot_size'), s.get('ms_per_step') and round(s['ms_per_step']*1000,1))" >> $O/bench.txt 2>&1; }
b c2 --steps 1000 --warmup 10
b c4 --config c4 --steps 50 --warmup 3 --no-shvs
b c5full --config c5 --variant full --steps 30 --warmup 3 --no-shvs
b c5shvs --config c5 --steps 30 --warmup 3
b c1 --config c1 --steps 1000 --warmup 10 --no-shvs
b c2long --config c2long --steps 100 --warmup 5 --no-shvs
echo done > $O/DONE
