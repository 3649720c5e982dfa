#!/bin/bash
# Alternating A/B of balanced vs greedy scoring passes on the C3 step.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
A="--steps 10 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for i in 1 2 3; do
  for m in greedy balanced; do
    timeout -s KILL 600 python scripts/ab_passes.py $m $A > gpurun_out/abp_${m}_$i.json 2>/dev/null
    echo -n "$m $i: "; python scripts/show.py gpurun_out/abp_${m}_$i.json | cut -c1-150
  done
done
