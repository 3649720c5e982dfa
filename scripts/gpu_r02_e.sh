#!/bin/bash
# Round 2, call E: full C3 step, G=3 (default) vs G=2 (pair MMA, weight-resident rasters),
# alternating runs on one box.
mkdir -p gpurun_out
for r in 1 2; do
  for g in 3 2; do
    KRR_GEMM_GEO=$g timeout 900 python bench.py --steps 5 --warmup 3 --latency-reps 0 --no-cpu-baseline --full-pairs 4 > gpurun_out/e_bench_g${g}_$r.log 2>&1
    tail -1 gpurun_out/e_bench_g${g}_$r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($g, $r, round(d['value'],1), d['clocks']['sm_mhz'], round(d['roofline']['achieved'],1), round(d['roofline']['gemm_share_of_step'],3))"
  done
done
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for shape in qkv wo up_store down; do
  for g in 3 2; do
    KRR_GEMM_GEO=$g timeout 300 ncu --metrics $M --clock-control none -k regex:gemm -s 3 -c 1 --csv python scripts/gemm_probe.py --shape $shape --reps 4 --m 307200 > gpurun_out/e_ncu_${shape}_g$g.csv 2>&1
    echo "$shape g$g $(grep -E 'dram__bytes_read|gpu__time|tensor|per_second' gpurun_out/e_ncu_${shape}_g$g.csv | awk -F'","' '{printf "%s ", $NF}')"
  done
done
