#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${1:-ab_persist}; mkdir -p $O
for v in ${VARIANTS:-default sw5 sw7}; do
  if [ $v = default ]; then L=""; else L=paper_2512_00719_b200/_lib/variants/$v.so; fi
  for spec in ${SPECS:-"c2 1000 0" "c2 20 0" "c4 30 4"}; do
    set -- $spec; c=$1; st=$2; fl=$3
    DP_LIB=$L timeout 900 python bench.py --config $c --steps $st --warmup 5 --no-cpu-baseline --no-shvs --plan-flags $fl 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $c steps $st flags $fl', round(d['ms_per_step']*1000,1), 'us', round(d['roofline']['frac'],3))" >> $O/ab.txt 2>&1
  done
done
