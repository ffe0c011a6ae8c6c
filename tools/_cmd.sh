cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests -m gpu -x -q -rs --durations=8 > gpurun_out/pytest_r2c.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2c.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_shvs_r2c.csv python tools/prof_step.py --variant shvs --steps 3 > /dev/null 2>&1
