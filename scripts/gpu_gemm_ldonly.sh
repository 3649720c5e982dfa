#!/bin/bash
# Diagnostic (timing only): G=8 epilogue that reads the accumulator from TMEM but skips the
# epilogue math and stores (_krr_ldonly.so) vs the full epilogue, ncu of the MLP-up launch.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for v in full ldonly; do
  L=""; [ $v = ldonly ] && L="KRR_LIB=$PWD/paper_2504_02921_b200/_krr_ldonly.so"
  for s in 2 1 0; do
    timeout -s KILL 900 env $L ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"gemm_tcgen05" -s $s -c 1 --csv $CMD > gpurun_out/ldo_${v}_$s.csv 2>/dev/null
    echo "$v s=$s rc=$?"; grep -E "gpu__time|tensor|per_second" gpurun_out/ldo_${v}_$s.csv | awk -F'","' '{print $(NF-2), $(NF)}' | tr -d '"'
  done
done
