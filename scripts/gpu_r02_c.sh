#!/bin/bash
# Round 2, call C: pair-MMA GEMM geometries (G=2, G=7) correctness + A/B vs G=3 and cuBLAS,
# with and without the cta_group::2 TMA (relay variant).
mkdir -p gpurun_out
P=paper_2504_02921_b200
for v in "default 2" "default 7" "relay 2" "relay 7"; do
  set -- $v
  lib=$P/_kvrerank_b200.so; [ $1 != default ] && lib=$P/_krr_$1.so
  KRR_LIB=$lib KRR_GEMM_GEO=$2 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k "gemm" -p no:cacheprovider > gpurun_out/c_t_$1_$2.log 2>&1
  echo "$v: $(tail -1 gpurun_out/c_t_$1_$2.log)"
done
for shape in up_store down; do
  for v in "default 3" "default 2" "default 7" "relay 2" "relay 7"; do
    set -- $v
    lib=$P/_kvrerank_b200.so; [ $1 != default ] && lib=$P/_krr_$1.so
    KRR_LIB=$lib KRR_GEMM_GEO=$2 timeout 120 python scripts/gemm_probe.py --shape $shape --reps 300 --tag "$1/$2" >> gpurun_out/c_gemm.jsonl 2>>gpurun_out/c_gemm.err
  done
  timeout 120 python scripts/gemm_probe.py --shape $shape --reps 300 --cublas --tag cublas >> gpurun_out/c_gemm.jsonl 2>>gpurun_out/c_gemm.err
done
cat gpurun_out/c_gemm.jsonl
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_ltcfabric.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for v in "default 7" "relay 2" "relay 7"; do
  set -- $v
  lib=$P/_kvrerank_b200.so; [ $1 != default ] && lib=$P/_krr_$1.so
  KRR_LIB=$lib KRR_GEMM_GEO=$2 timeout 300 ncu --metrics $M --clock-control none -k regex:gemm -s 3 -c 1 --csv python scripts/gemm_probe.py --shape up_store --reps 4 --m 307200 > gpurun_out/c_ncu_$1_$2.csv 2>&1
done
for f in gpurun_out/c_ncu_*.csv; do echo $f; grep -E "dram__bytes_read|ltcfabric|gpu__time|tensor|per_second" $f | awk -F'","' '{print $(NF-2), $NF}'; done
