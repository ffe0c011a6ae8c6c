cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r3t; mkdir -p $O
for v in default rank200 rank640; do
  if [ $v = default ]; then L=""; else L=paper_2512_00719_b200/_lib/variants/$v.so; fi
  for c in c2 c4 c2long; do
    st=300; [ $c = c4 ] && st=30; [ $c = c2long ] && st=50
    DP_LIB=$L timeout 600 python bench.py --config $c --steps $st --warmup 5 --no-cpu-baseline --no-shvs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', round(d['ms_per_step']*1000,1), 'us', round(d['roofline']['frac'],3))" >> $O/ab.txt 2>&1
  done
done
