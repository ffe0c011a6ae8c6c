#!/bin/bash
# parity + the five configs' full-path steps (one line each)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${1:-q5}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -rs -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
for spec in "c2 1000" "c2 20" "c4 30" "c5 20" "c1 300" "c2long 50"; do
  set -- $spec; c=$1; st=$2
  var=""; [ $c = c5 ] && var="--variant full"
  timeout 900 python bench.py --config $c $var --steps $st --warmup 5 --no-cpu-baseline --no-shvs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $st', round(d['ms_per_step']*1000,1), 'us', round(d['roofline']['frac'],3))" >> $O/ab.txt 2>&1
done
