#!/bin/bash
# One GPU round-trip producing the round's evidence:
#   parity tests, smoke, bench lines (full + SHVS + reference arm), the ncu
#   launch list of the bench command and one `ncu --set full` capture of the
#   dominant kernel.  usage: tools/gpu_full.sh TAG
TAG=${1:-r1}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -rs --durations=8 > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 600 python bench.py > $O/bench_c2_full.jsonl 2> $O/bench_c2_full.err
timeout 600 python bench.py --variant shvs --no-cpu-baseline > $O/bench_c2_shvs.jsonl 2> $O/bench_c2_shvs.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.jsonl 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2_full.csv \
  python bench.py --steps 2 --warmup 3 --kernel-steps 2 --no-cpu-baseline > $O/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"topk_sample|stream_sample|general" -s 2 -c 1 \
  -o $O/full_c2 python tools/prof_step.py --steps 4 > $O/ncu_full_c2.log 2>&1
ncu -i $O/full_c2.ncu-rep --page raw --csv > $O/full_c2_raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"shvs|warp|topk_sample" -s 4 -c 2 \
  -o $O/full_shvs python tools/prof_step.py --variant shvs --steps 4 > $O/ncu_full_shvs.log 2>&1
ncu -i $O/full_shvs.ncu-rep --page raw --csv > $O/full_shvs_raw.csv 2>/dev/null
echo done > $O/DONE
