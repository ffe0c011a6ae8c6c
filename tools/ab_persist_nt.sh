cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-r4l}; mkdir -p $O
for v in ${VARIANTS:-default nt288 nt320 nt384}; do
  if [ $v = default ]; then L=""; else L=paper_2512_00719_b200/_lib/variants/$v.so; fi
  for st in 1000 20; do
    DP_LIB=$L timeout 900 python bench.py --config c2 --steps $st --warmup 5 --no-cpu-baseline --no-shvs --plan-flags 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c2 steps $st', round(d['ms_per_step']*1000,1), 'us', round(d['roofline']['frac'],3))" >> $O/ab.txt 2>&1
  done
done
