cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/b4; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -rs > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
bash tools/bench_all.sh b4
for c in c2p c2m c2n; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --steps 50 --warmup 3 > $O/bench_$c.jsonl 2>$O/bench_$c.err
done
timeout 900 python tools/c3_sweep.py --out $O/c3_sweep.json > $O/c3.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2_full.csv python bench.py --steps 2 --warmup 3 --kernel-steps 2 --no-cpu-baseline --no-shvs > $O/ncu_launch.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2_shvs.csv python bench.py --variant shvs --steps 2 --warmup 3 --kernel-steps 2 --no-cpu-baseline > $O/ncu_launch2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"topk_sample" -s 2 -c 1 -o $O/full_c2 python tools/prof_step.py --steps 4 > $O/ncu_full_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"warp_sample|topk_sample" -s 2 -c 2 -o $O/full_shvs python tools/prof_step.py --variant shvs --steps 4 > $O/ncu_full_shvs.log 2>&1
