#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for cfg in "KRR_GEMM_RASTER=m" "KRR_GEMM_RASTER=n" "KRR_GEMM_GROUP_M=4" "KRR_GEMM_GROUP_M=16" "KRR_GEMM_CTA=1"; do
  echo "== $cfg"
  env $cfg timeout -s KILL 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:gemm_tcgen05 -s 1 -c 1 --csv python scripts/gemm_traffic.py 2>/dev/null | grep -E "dram__|gpu__time|lts__" | awk -F'","' '{print "   " $(NF-2) " " $(NF-1) " " $NF}'
done
