#!/bin/bash
# Round 2, first call: GPU test suite after the ownership/pruning changes, GEMM
# cache-hint A/B (mode 4 vs cta_group::2 mode 2), and a default bench line.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/a_gpu.txt
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/a_tests.log 2>&1
tail -30 gpurun_out/a_tests.log
P=paper_2504_02921_b200
for shape in up_store down; do
  for v in "default 4" "default 2" "h1 2" "h2 2" "h1 4"; do
    set -- $v
    lib=$P/_kvrerank_b200.so; [ $1 != default ] && lib=$P/_krr_$1.so
    KRR_LIB=$lib KRR_GEMM_CTA=$2 timeout 120 python scripts/gemm_probe.py --shape $shape --reps 200 --tag "$1/$2" >> gpurun_out/a_gemm.jsonl 2>>gpurun_out/a_gemm.err
  done
  timeout 120 python scripts/gemm_probe.py --shape $shape --reps 200 --cublas --tag cublas >> gpurun_out/a_gemm.jsonl 2>>gpurun_out/a_gemm.err
done
for v in "default 4" "default 2" "h1 2" "h2 2" "h1 4"; do
  set -- $v
  lib=$P/_kvrerank_b200.so; [ $1 != default ] && lib=$P/_krr_$1.so
  KRR_LIB=$lib KRR_GEMM_CTA=$2 timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_ltcfabric.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gemm -s 3 -c 1 --csv python scripts/gemm_probe.py --shape up_store --reps 4 --m 307200 > gpurun_out/a_ncu_$1_$2.csv 2>&1
done
timeout 900 python bench.py > gpurun_out/a_bench.log 2>&1
tail -3 gpurun_out/a_bench.log
cat gpurun_out/a_gemm.jsonl
