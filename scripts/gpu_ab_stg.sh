#!/bin/bash
# G=8 epilogue: 16-bit chunks double-buffered in the warp's 4 KB staging (default) vs the
# single-buffered variant (_krr_stg1.so, built from the previous source), C3 step, alternating.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -q -m gpu -k "gemm or parity" --timeout 600 -p no:cacheprovider > gpurun_out/abs_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED" gpurun_out/abs_pytest.log | tail -4
A="--steps 10 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for i in 1 2 3; do
  timeout -s KILL 600 env KRR_LIB=$PWD/paper_2504_02921_b200/_krr_stg1.so python bench.py $A > gpurun_out/abs_stg1_$i.json 2>/dev/null
  echo -n "stg1 $i: "; python scripts/show.py gpurun_out/abs_stg1_$i.json | cut -c1-150
  timeout -s KILL 600 python bench.py $A > gpurun_out/abs_stg2_$i.json 2>/dev/null
  echo -n "stg2 $i: "; python scripts/show.py gpurun_out/abs_stg2_$i.json | cut -c1-150
done
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for v in stg2 stg1; do
  L=""; [ $v = stg1 ] && L="KRR_LIB=$PWD/paper_2504_02921_b200/_krr_stg1.so"
  timeout -s KILL 900 env $L ncu --nvtx --nvtx-include "timed/" --set full --clock-control none -k regex:"gemm_tcgen05" -s 2 -c 1 -o gpurun_out/abs_${v}_gemm $CMD > /dev/null 2>&1
  echo "ncu $v rc=$?"
done
