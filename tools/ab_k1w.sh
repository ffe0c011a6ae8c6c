#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${1:-ab_k1w}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "shvs" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
for v in default u8; do
  if [ $v = default ]; then L=""; else L=paper_2512_00719_b200/_lib/variants/$v.so; fi
  for c in c2 c3; do
    DP_LIB=$L timeout 900 python bench.py --config $c --variant shvs --steps 300 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $c shvs', round(d['ms_per_step']*1000,1), 'us H', d['config']['hot_size'], 'kern', round(d['roofline']['kernel_ms']*1000,1))" >> $O/ab.txt 2>&1
  done
done
