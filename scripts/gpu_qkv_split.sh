#!/bin/bash
# Diagnostic (timing only): QKV epilogue without RoPE math (_krr_norope.so) or without the
# global stores (_krr_nostore.so) vs the full epilogue; ncu of the first QKV launch of the C3 step.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for v in full norope nostore; do
  L=""; [ $v != full ] && L="KRR_LIB=$PWD/paper_2504_02921_b200/_krr_$v.so"
  timeout -s KILL 900 env $L ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"gemm_tcgen05" -s 0 -c 1 --csv $CMD > gpurun_out/qs_${v}.csv 2>/dev/null
  echo -n "$v rc=$? "; grep -E '^"[0-9]' gpurun_out/qs_${v}.csv | python3 -c "
import csv,sys
v=[float(r[-1].replace(',','')) for r in csv.reader(sys.stdin)]
print(f'time {v[0]/1e6:.3f} ms clock {v[1]/1e9:.3f} GHz cycles {v[0]*v[1]/1e15:.3f} M')"
done
