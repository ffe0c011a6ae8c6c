cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/it32; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
for args in "--config c5 --steps 30" "--config c2n --steps 50" "--config c2p --steps 50" "--config c2m --steps 50"; do
  echo "$args" >> $O/bench.txt
  timeout 300 python bench.py --no-cpu-baseline --no-shvs --warmup 3 $args 2>>$O/err.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])" >> $O/bench.txt 2>&1
done
