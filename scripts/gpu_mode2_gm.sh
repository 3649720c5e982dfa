#!/bin/bash
# cta_group::2 (mode 2) raster group sweep: DRAM/L2 misses (ncu) and sustained clocks
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for gm in 2 4 8 16; do
  echo "== CTA=2 GROUP_M=$gm"
  KRR_GEMM_CTA=2 KRR_GEMM_GROUP_M=$gm timeout -s KILL 600 ncu --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_ltcfabric.sum --clock-control none -k regex:gemm_tcgen05 -s 1 -c 1 --csv python scripts/gemm_traffic.py 2>/dev/null | grep -E "dram__|gpu__time|lts__" | awk -F'","' '{print "   " $(NF-2) " " $(NF-1) " " $NF}'
done
echo "== CTA=4 GROUP_M=8"
KRR_GEMM_CTA=4 timeout -s KILL 600 ncu --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_ltcfabric.sum --clock-control none -k regex:gemm_tcgen05 -s 1 -c 1 --csv python scripts/gemm_traffic.py 2>/dev/null | grep -E "dram__|gpu__time|lts__" | awk -F'","' '{print "   " $(NF-2) " " $(NF-1) " " $NF}'
