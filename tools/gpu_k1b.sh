cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r4o; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -rs -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5_shvs.csv python tools/prof_step.py --config c5 --variant shvs --hot 2048 --steps 2 --extra fused > /dev/null 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2n.csv python tools/prof_step.py --config c2n --steps 2 > /dev/null 2>&1
python tools/ncu_summary.py $O > $O/summary.md
for c in c5 c2n c2p; do timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-shvs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['config']['variant'], round(d['ms_per_step']*1000,1), 'us')" >> $O/ab.txt; done
timeout 900 python bench.py --config c5 --variant full --steps 20 --warmup 3 --no-cpu-baseline --no-shvs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 full', round(d['ms_per_step']*1000,1), 'us')" >> $O/ab.txt
