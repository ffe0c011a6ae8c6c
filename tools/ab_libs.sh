#!/bin/bash
# A-B of library variants on the bench configs: bash tools/ab_libs.sh TAG lib1 lib2 ...
# (paths relative to the repo; "default" = the in-tree build)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=$1; shift
O=gpurun_out/$TAG; mkdir -p $O
b() { local lib=$1 n=$2; shift 2; local env=""; [ "$lib" != default ] && env="DP_LIB=$lib";
  env $env timeout 600 python bench.py "$@" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d.get('shvs') or {}; print('$(basename $lib)', '$n', round(d['ms_per_step']*1000,1), 'us frac', round(d['roofline']['frac'],3), 'shvs', s.get('hot_size'), s.get('ms_per_step') and round(s['ms_per_step']*1000,1))" >> $O/ab.txt 2>&1; }
for rep in 1 2; do
  for lib in "$@"; do
    b $lib c2 --steps 1000 --warmup 10
    b $lib c4 --config c4 --steps 50 --warmup 3 --no-shvs
    b $lib c1 --config c1 --steps 1000 --warmup 10 --no-shvs
  done
done
echo done > $O/DONE
