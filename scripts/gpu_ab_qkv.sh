#!/bin/bash
# QKV epilogue: per-row async bulk copies (default) vs LSU stores through a transposed
# staging buffer (_krr_qkvold.so): GPU tests, ncu of the first QKV launch, C3 step A/B.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/abq_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^ERROR" gpurun_out/abq_pytest.log | tail -6
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for v in new old; do
  L=""; [ $v = old ] && L="KRR_LIB=$PWD/paper_2504_02921_b200/_krr_qkvold.so"
  timeout -s KILL 900 env $L ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"gemm_tcgen05" -s 0 -c 1 --csv $CMD > gpurun_out/abq_${v}_ncu.csv 2>/dev/null
  echo "ncu $v rc=$?"; grep -E '^"[0-9]' gpurun_out/abq_${v}_ncu.csv | python3 -c "
import csv,sys
for r in csv.reader(sys.stdin): print('  ', r[-3], r[-1])"
done
A="--steps 10 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for i in 1 2; do
  timeout -s KILL 600 env KRR_LIB=$PWD/paper_2504_02921_b200/_krr_qkvold.so python bench.py $A > gpurun_out/abq_old_$i.json 2>/dev/null
  echo -n "old $i: "; python scripts/show.py gpurun_out/abq_old_$i.json | cut -c1-150
  timeout -s KILL 600 python bench.py $A > gpurun_out/abq_new_$i.json 2>/dev/null
  echo -n "new $i: "; python scripts/show.py gpurun_out/abq_new_$i.json | cut -c1-150
done
