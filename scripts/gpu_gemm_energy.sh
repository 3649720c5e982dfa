#!/bin/bash
# sustained GEMM energy per FLOP by mode (gemm_bench, 200 reps per shape, nvidia-smi sampling)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for cta in 4 1 2; do
  echo "== CTA=$cta"
  KRR_GEMM_CTA=$cta timeout -s KILL 900 python scripts/gemm_bench.py --m 65536 --reps 200 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    l = l.strip()
    if l.startswith('{'):
        d = json.loads(l)
        for k, v in d.items():
            if isinstance(v, dict) and 'ms' in v and k in ('up_gelu', 'up_store', 'up_store_cublas', 'down', 'down_cublas'):
                tf, w, mhz = v['tflops'], v['watts'], v['sm_mhz']
                print(f'   {k:16s} {tf:7.1f} TF/s  {mhz:6.0f} MHz  {w:6.0f} W  {tf/w*1000 if w else 0:6.1f} GF/J  {tf*1e3/(148*mhz) if mhz else 0:6.0f} FLOP/clk/SM')
"
done
