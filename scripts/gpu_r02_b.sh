#!/bin/bash
# Round 2, call B: full GPU suite (drop-in forward, C5/top-k/bf16 parity, ownership),
# bench --gpus 2 self-launch on one GPU (gloo), the reference arm, GEMM mode-2 raster probe.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider -rf > gpurun_out/b_tests.log 2>&1
tail -40 gpurun_out/b_tests.log
KRR_BENCH_ONE_DEVICE=1 KRR_BENCH_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --latency-reps 2 --full-pairs 4 > gpurun_out/b_bench2.log 2>&1
tail -2 gpurun_out/b_bench2.log | cut -c1-600
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/b_ref.log 2>&1
tail -1 gpurun_out/b_ref.log | cut -c1-400
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_ltcfabric.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__cluster_dim_x"
for v in "4 8" "2 8" "2 4" "2 16" "2 32"; do
  set -- $v
  KRR_GEMM_CTA=$1 KRR_GEMM_GROUP_M=$2 timeout 300 ncu --metrics $M --clock-control none -k regex:gemm -s 3 -c 1 --csv python scripts/gemm_probe.py --shape up_store --reps 4 --m 307200 > gpurun_out/b_ncu_m$1_g$2.csv 2>&1
done
for f in gpurun_out/b_ncu_*.csv; do echo $f; grep -E "dram__bytes_read|grid_size|ltcfabric|gpu__time" $f | awk -F'","' '{print $(NF-2), $NF}'; done
