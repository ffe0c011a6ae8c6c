cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/it25; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
for c in c2 c4 c2p; do
  echo "$c" >> $O/bench.txt
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-shvs --steps 100 --warmup 3 2>>$O/err.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])" >> $O/bench.txt 2>&1
done
