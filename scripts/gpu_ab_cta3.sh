#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for i in 1 2; do for c in 1 3; do
  KRR_GEMM_CTA=$c timeout -s KILL 600 $B > gpurun_out/ab3_cta${c}_$i.json 2>/dev/null
  echo -n "cta=$c run=$i "; tail -1 gpurun_out/ab3_cta${c}_$i.json | python scripts/show.py
done; done
