#!/bin/bash
# Round 2, call D: why the pair geometries read 3-5x the DRAM of G=3 (ncu --set full
# side by side), N-band rasters for the pair geometries, and the full C3 step per geometry.
mkdir -p gpurun_out
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_ltcfabric.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for v in "3 8" "2 -16" "2 -8" "7 -16" "7 -8" "7 2" "7 8"; do
  set -- $v
  KRR_GEMM_GEO=$1 KRR_GEMM_GROUP_M=$2 timeout 300 ncu --metrics $M --clock-control none -k regex:gemm -s 3 -c 1 --csv python scripts/gemm_probe.py --shape up_store --reps 4 --m 307200 > gpurun_out/d_ncu_g$1_m$2.csv 2>&1
done
for f in gpurun_out/d_ncu_*.csv; do echo $f; grep -E "dram__bytes_read|ltcfabric|gpu__time|tensor|per_second" $f | awk -F'","' '{print $(NF-2), $NF}'; done
for g in 3 2; do
  KRR_GEMM_GEO=$g timeout 300 ncu --set full --clock-control none -k regex:gemm -s 3 -c 1 -o gpurun_out/d_full_g$g python scripts/gemm_probe.py --shape up_store --reps 4 --m 65536 > gpurun_out/d_full_g$g.log 2>&1
done
for g in 3 7; do
  KRR_GEMM_GEO=$g timeout 900 python bench.py --steps 5 --warmup 3 --latency-reps 0 --no-cpu-baseline --full-pairs 4 > gpurun_out/d_bench_g$g.log 2>&1
  tail -1 gpurun_out/d_bench_g$g.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($g, d['value'], d['clocks'], d['roofline']['achieved'])"
done
