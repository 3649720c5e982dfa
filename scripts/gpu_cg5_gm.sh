#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for gm in 2 4 8 16; do
  echo "== CTA=6 GROUP_M=$gm"
  KRR_GEMM_CTA=6 KRR_GEMM_GROUP_M=$gm timeout -s KILL 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none -k regex:gemm_tcgen05 -s 1 -c 1 --csv python scripts/gemm_traffic.py 2>/dev/null | grep -E "dram__|gpu__time|tensor|per_second|hit_rate" | awk -F'","' '{print "   " $(NF-2) " " $(NF-1) " " $NF}'
done
