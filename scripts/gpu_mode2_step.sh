#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for i in 1 2; do for cfg in "4 8" "2 16" "2 32"; do
  set -- $cfg
  KRR_GEMM_CTA=$1 KRR_GEMM_GROUP_M=$2 timeout -s KILL 600 $B > gpurun_out/m2s_${1}_${2}_$i.json 2>/dev/null
  echo -n "cta=$1 gm=$2 run=$i "; tail -1 gpurun_out/m2s_${1}_${2}_$i.json | python scripts/show.py
done; done
