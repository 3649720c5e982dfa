#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for cta in 4 2; do
  echo "== gemm_bench CTA=$cta M=65536"
  KRR_GEMM_CTA=$cta timeout -s KILL 600 python scripts/gemm_bench.py --m 65536 --reps 30 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    l = l.strip()
    if l.startswith('{'):
        d = json.loads(l)
        print('  ', {k: (v['ms'], v['tflops'], v['sm_mhz'], v['watts']) for k, v in d.items() if isinstance(v, dict) and 'ms' in v})
"
done
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for i in 1 2; do for cta in 4 2; do
  KRR_GEMM_CTA=$cta timeout -s KILL 600 $B > gpurun_out/cta2_${cta}_$i.json 2>/dev/null
  echo -n "cta=$cta run=$i "; tail -1 gpurun_out/cta2_${cta}_$i.json | python scripts/show.py
done; done
