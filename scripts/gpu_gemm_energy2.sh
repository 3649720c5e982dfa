#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
P=$PWD/paper_2504_02921_b200
for v in default noepi default noepi; do
  lib=$P/_krr_$v.so; [ "$v" = default ] && lib=$P/_kvrerank_b200.so
  echo "== $v"
  KRR_LIB=$lib timeout -s KILL 900 python scripts/gemm_bench.py --m 65536 --reps 200 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    l = l.strip()
    if l.startswith('{'):
        d = json.loads(l)
        for k, v in d.items():
            if isinstance(v, dict) and 'ms' in v and k in ('up_store', 'down', 'qkv'):
                tf, w, mhz = v['tflops'], v['watts'], v['sm_mhz']
                print(f'   {k:16s} {tf:7.1f} TF/s  {mhz:6.0f} MHz  {w:6.0f} W  {tf/w*1000 if w else 0:6.1f} GF/J')
"
done
