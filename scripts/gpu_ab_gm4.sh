#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for i in 1 2; do for gm in 8 4 16; do
  KRR_GEMM_GROUP_M=$gm timeout -s KILL 600 $B > gpurun_out/abgm4_${gm}_$i.json 2>/dev/null
  echo -n "gm=$gm run=$i "; tail -1 gpurun_out/abgm4_${gm}_$i.json | python scripts/show.py
done; done
