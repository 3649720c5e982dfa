#!/bin/bash
# GEMM geometry DRAM probe (variant library from an older tree under _var/, env KRR_GEMM_GEO).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_ltcfabric.sum,sm__cycles_elapsed.avg.per_second,launch__grid_size"
for shape in up_store qkv; do
  for geo in 3 2; do
    (cd _var && KRR_GEMM_GEO=$geo timeout 300 ncu --metrics $M --clock-control none -k regex:gemm -s 3 -c 1 --csv python scripts/gemm_probe.py --shape $shape --reps 4 --m 65536) > gpurun_out/g2p_${shape}_$geo.csv 2>&1
    echo "== $shape geo=$geo"; grep -E '"(dram__|gpu__time|lts__|sm__cycles|launch__grid)' gpurun_out/g2p_${shape}_$geo.csv | awk -F'","' '{printf "   %-60s %s %s\n", $(NF-2), $(NF-1), $NF}'
  done
done
