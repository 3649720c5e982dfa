#!/bin/bash
# Alternating full-step A/B between this tree and an older checkout under _ab_old/
# (git archive + build; not committed).  usage: gpurun -- bash scripts/gpu_ab_tree.sh TAG ROUNDS [bench args]
TAG=${1:-ab}; N=${2:-2}; shift 2
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for i in $(seq $N); do
  for side in new old; do
    d=.; [ $side = old ] && d=_ab_old
    (cd $d && timeout -s KILL 600 python bench.py --steps 3 --warmup 2 --latency-reps 0 --full-pairs 4 --no-cpu-baseline "$@") > gpurun_out/${TAG}_${side}_$i.json 2> gpurun_out/${TAG}_${side}_$i.err
    echo -n "$side $i: "; python scripts/show.py gpurun_out/${TAG}_${side}_$i.json
  done
done
