#!/bin/bash
# energy decomposition: operand movement only (MMA off) vs full, mode 4 vs mode 2
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
P=$PWD/paper_2504_02921_b200
for r in 1 2; do for v in default nomma; do for cta in 4 2; do
  lib=$P/_krr_$v.so; [ "$v" = default ] && lib=$P/_kvrerank_b200.so
  echo -n "$v cta=$cta run=$r: "
  KRR_LIB=$lib KRR_GEMM_CTA=$cta timeout -s KILL 600 python scripts/gemm_bench.py --m 65536 --reps 300 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    l = l.strip()
    if l.startswith('{'):
        d = json.loads(l); v = d['up_store']
        print(f\"up_store {v['ms']:.3f} ms  {v['sm_mhz']:.0f} MHz  {v['watts']:.0f} W\")
"
done; done; done
