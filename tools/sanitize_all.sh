#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on tools/sanitize.py
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${1:-san}; mkdir -p $O
for t in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py > $O/$t.txt 2>&1
  echo "rc=$?" >> $O/$t.txt
done
