#!/bin/bash
# A-B of the admission-estimate factor (DP_EST_OVER) across configs
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${1:-ab_est}; mkdir -p $O
for v in default est2 est3; do
  if [ $v = default ]; then L=""; else L=paper_2512_00719_b200/_lib/variants/$v.so; fi
  for spec in "c2 1000" "c4 30" "c5 20" "c1 300" "c2long 50"; do
    set -- $spec; c=$1; st=$2
    var=""; [ $c = c5 ] && var="--variant full"
    DP_LIB=$L timeout 900 python bench.py --config $c $var --steps $st --warmup 5 --no-cpu-baseline --no-shvs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', round(d['ms_per_step']*1000,1), 'us', round(d['roofline']['frac'],3))" >> $O/ab.txt 2>&1
  done
done
