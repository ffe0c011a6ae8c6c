#!/bin/bash
# The round's final evidence in one GPU call: parity + smoke, every bench
# line (incl. the reference arm), the ncu capture of every kernel, sanitizers.
TAG=${1:-final}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=10 > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
bash tools/bench_all.sh ${TAG}_bench
bash tools/ncu_all.sh ${TAG}_ncu
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py > $O/$t.txt 2>&1; echo "rc=$?" >> $O/$t.txt
done
echo done > $O/DONE
