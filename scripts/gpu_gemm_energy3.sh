#!/bin/bash
# energy per FLOP vs raster group size, cta_group::2 (mode 2) and multicast (mode 4)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for cfg in "2 8" "2 32" "4 8" "4 32"; do
  set -- $cfg
  echo "== CTA=$1 GROUP_M=$2"
  KRR_GEMM_CTA=$1 KRR_GEMM_GROUP_M=$2 timeout -s KILL 900 python scripts/gemm_bench.py --m 65536 --reps 200 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    l = l.strip()
    if l.startswith('{'):
        d = json.loads(l)
        for k, v in d.items():
            if isinstance(v, dict) and 'ms' in v and k in ('up_store', 'down', 'up_store_cublas'):
                tf, w, mhz = v['tflops'], v['watts'], v['sm_mhz']
                print(f'   {k:16s} {tf:7.1f} TF/s  {mhz:6.0f} MHz  {w:6.0f} W  {tf/w*1000 if w else 0:6.1f} GF/J')
"
done
