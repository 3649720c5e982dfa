#!/bin/bash
# QKV epilogue: RoPE cos/sin loaded before the chunk's TMEM read (default) vs after it
# (_krr_ropeold.so): GEMM/parity tests, ncu of the first QKV launch, C3 step A/B.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/abr_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^ERROR" gpurun_out/abr_pytest.log | tail -6
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for v in new old; do
  L=""; [ $v = old ] && L="KRR_LIB=$PWD/paper_2504_02921_b200/_krr_ropeold.so"
  timeout -s KILL 900 env $L ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"gemm_tcgen05" -s 0 -c 1 --csv $CMD > gpurun_out/abr_${v}.csv 2>/dev/null
  echo -n "ncu $v rc=$? "; grep -E '^"[0-9]' gpurun_out/abr_${v}.csv | python3 -c "
import csv,sys
v=[float(r[-1].replace(',','')) for r in csv.reader(sys.stdin)]
print(f'time {v[0]/1e6:.3f} ms clock {v[1]/1e9:.3f} GHz cycles {v[0]*v[1]/1e15:.3f} M')"
done
A="--steps 10 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for i in 1 2; do
  timeout -s KILL 600 env KRR_LIB=$PWD/paper_2504_02921_b200/_krr_ropeold.so python bench.py $A > gpurun_out/abr_old_$i.json 2>/dev/null
  echo -n "old $i: "; python scripts/show.py gpurun_out/abr_old_$i.json | cut -c1-150
  timeout -s KILL 600 python bench.py $A > gpurun_out/abr_new_$i.json 2>/dev/null
  echo -n "new $i: "; python scripts/show.py gpurun_out/abr_new_$i.json | cut -c1-150
done
