#!/bin/bash
# GROUP_M fixed 8 vs per-K auto: MLP-up / down traffic (ncu) and the C3 step, alternating
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for i in 1 2 3; do for gm in 8 auto; do
  KRR_GEMM_GROUP_M=$gm timeout -s KILL 600 $B > gpurun_out/gma_${gm}_$i.json 2>/dev/null
  echo -n "gm=$gm run=$i "; tail -1 gpurun_out/gma_${gm}_$i.json | python scripts/show.py
done; done
