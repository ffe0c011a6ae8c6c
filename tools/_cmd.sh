cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/it15; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
DP_LIB=paper_2512_00719_b200/_lib/variants/prof.so python tools/phase_prof.py --variant shvs > $O/phase.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 200 --variant shvs 2>>$O/err.txt | tail -1 > $O/bench_shvs.jsonl
