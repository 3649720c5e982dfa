#!/bin/bash
# GEMM geometry DRAM probe at the full C3 MLP-up M (variant tree under _var/, env KRR_GEMM_GEO / GROUP_M).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,sm__cycles_elapsed.avg.per_second"
for v in "3 8" "2 8" "3 -8" "2 -8" "2 -4" "2 4"; do
  set -- $v
  (cd _var && KRR_GEMM_GEO=$1 KRR_GEMM_GROUP_M=$2 timeout 300 ncu --metrics $M --clock-control none -k regex:gemm -s 2 -c 1 --csv python scripts/gemm_probe.py --shape up_store --reps 3 --m 307200) > gpurun_out/g2q_$1_$2.csv 2>&1
  echo "== geo=$1 group_m=$2 $(grep -E '"(dram__|gpu__time|lts__|sm__cycles)' gpurun_out/g2q_$1_$2.csv | awk -F'","' '{printf "%s=%s ", $(NF-2), $NF}')"
done
