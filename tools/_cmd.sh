cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/it33; mkdir -p $O
timeout 600 python bench.py --no-cpu-baseline --steps 500 > $O/c2.jsonl 2>$O/err.txt
timeout 600 python bench.py --no-cpu-baseline --steps 500 --hot 2048 > $O/c2_h2k.jsonl 2>>$O/err.txt
timeout 600 python bench.py --no-cpu-baseline --steps 500 --hot 8192 > $O/c2_h8k.jsonl 2>>$O/err.txt
