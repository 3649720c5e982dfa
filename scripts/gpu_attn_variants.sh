#!/bin/bash
# attention micro-benchmark across variant libraries (KRR_LIB), interleaved
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
P=$PWD/paper_2504_02921_b200
for r in 1 2; do for v in "$@"; do
  lib=$P/_krr_$v.so; [ "$v" = default ] && lib=$P/_kvrerank_b200.so
  echo "== $v (run $r)"; KRR_LIB=$lib python scripts/attn_bench.py --pairs 6400 --boost 1 16 --backends tc --reps 30 2>&1 | tail -2
done; done
