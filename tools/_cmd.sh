cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/it26; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
for c in c2 c4 c3 c2p; do
  echo "$c" >> $O/bench.txt
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-shvs --steps 100 --warmup 3 2>>$O/err.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])" >> $O/bench.txt 2>&1
done
echo shvs >> $O/bench.txt
timeout 300 python bench.py --variant shvs --no-cpu-baseline --steps 200 2>>$O/err.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], d['roofline']['kernel_ms'])" >> $O/bench.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"topk_sample" -s 2 -c 1 -o $O/full_c2 python tools/prof_step.py --steps 4 > $O/ncu_full_c2.log 2>&1
