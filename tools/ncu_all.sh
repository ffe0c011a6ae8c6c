#!/bin/bash
# One `ncu --set full` capture per decision-plane kernel (one launch each),
# plus the launch list of the C2 bench step; summaries -> gpurun_out/$TAG.
#   tools/ncu_all.sh TAG
TAG=${1:-ncu}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/$TAG; mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
cap() {   # name kernel-regex (on the mangled name) skip args...
  local name=$1 k=$2 s=$3; shift 3
  timeout 300 $NCU --kernel-name-base mangled -k regex:$k -s $s -c 1 -o $O/$name python tools/prof_step.py "$@" \
    > $O/$name.log 2>&1
}
cap k1p_c2      topk_persist   1 --config c2 --steps 3
cap k1_c4       topk_sample    1 --config c4 --steps 2
cap k1w_hot_c2  warp_sample    1 --config c2 --variant shvs --hot 2048 --steps 3
cap k1_tail_c2  'topk_sample_kernelIfLi2E' 1 --config c2 --variant shvs --hot 2048 --steps 3
cap k1b_c2n     general_sample 1 --config c2n --steps 3
cap k2_raw_c2   'row_summary_kernelIfLi256ELi4ELb0E' 0 --config c2 --variant shvs --hot 2048 --steps 1
cap k2_pen_c2   'row_summary_kernelIfLi256ELi4ELb1E' 0 --config c2 --variant shvs --hot 2048 --steps 1 --extra summary
cap k6_c2       hot_mass_curve 0 --config c2 --variant shvs --hot 32768 --steps 1 --extra curve
cap synth_fused synth_summary  0 --config c2 --variant shvs --hot 2048 --steps 1 --extra fused
cap k1w_hot_c5  warp_sample    1 --config c5 --variant shvs --hot 2048 --steps 2
cap k1_c5_full  topk_sample    1 --config c5 --steps 2
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/launches_c2_full.csv python tools/prof_step.py --config c2 --steps 4 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/launches_c2_shvs.csv python tools/prof_step.py --config c2 --variant shvs --hot 2048 \
  --extra fused --steps 4 > /dev/null 2>&1
python tools/ncu_summary.py $O > $O/summary.md 2>&1
# keep the reports under gpurun's 64 MiB return limit: raw metric dumps for all,
# the full report only for the headline kernel
for r in $O/*.ncu-rep; do ncu -i $r --page raw --csv > ${r%.ncu-rep}.raw.csv 2>/dev/null; done
for r in $O/*.ncu-rep; do case $r in *k1p_c2*) ;; *) rm -f $r ;; esac; done
echo done > $O/DONE
