cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/it22; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -rs > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
for c in c2p c2m c2n; do
  echo "$c" >> $O/bench.txt
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-shvs --steps 50 --warmup 3 2>>$O/err.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])" >> $O/bench.txt 2>&1
done
timeout 600 python bench.py --config c5 --steps 50 --warmup 3 --no-cpu-baseline > $O/bench_c5.jsonl 2> $O/err_c5.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv python tools/prof_step.py --config c5 --variant shvs --steps 2 > $O/ncu_c5.log 2>&1
