cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2y; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -rs --durations=10 > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
bash tools/bench_all.sh r2y
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base mangled"
for spec in "k1_tail_c2 topk_sample_kernelIfLi2E 1 --config c2 --variant shvs --hot 2048 --steps 3" \
            "k2_raw_c2 row_summary_kernelIfLi256ELi4ELb0E 0 --config c2 --variant shvs --hot 2048 --steps 1" \
            "k2_pen_c2 row_summary_kernelIfLi256ELi4ELb1E 0 --config c2 --variant shvs --hot 2048 --steps 1 --extra summary"; do
  set -- $spec; name=$1; k=$2; s=$3; shift 3
  timeout 300 $NCU -k regex:$k -s $s -c 1 -o $O/$name python tools/prof_step.py "$@" > $O/$name.log 2>&1
done
python tools/ncu_summary.py $O > $O/ncu_summary.md 2>&1
for r in $O/*.ncu-rep; do ncu -i $r --page raw --csv > ${r%.ncu-rep}.raw.csv 2>/dev/null; rm -f $r; done
echo done > $O/DONE
