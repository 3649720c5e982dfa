#!/bin/bash
# GEMM tile-width sweep at the per-query latency batch (M = 100 pairs x 48 rows)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for M in 4800 9600; do for cta in 4 1; do for bn in 256 128 64; do
  echo "== M=$M cta=$cta bn=$bn"
  KRR_GEMM_CTA=$cta KRR_GEMM_BN=$bn timeout -s KILL 300 python scripts/gemm_bench.py --m $M --reps 50 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    l = l.strip()
    if l.startswith('{'):
        d = json.loads(l)
        print('  ', {k: (v['ms'], v['tflops'], v['sm_mhz']) for k, v in d.items() if isinstance(v, dict) and 'ms' in v})
"
done; done; done
