#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
KRR_GEMM_CTA=5 timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -1
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for i in 1 2; do for c in 4 5 1; do
  KRR_GEMM_CTA=$c timeout -s KILL 600 $B > gpurun_out/abmc2_cta${c}_$i.json 2>gpurun_out/abmc2_cta${c}_$i.err
  echo -n "cta=$c run=$i "; tail -1 gpurun_out/abmc2_cta${c}_$i.json | python scripts/show.py; tail -1 gpurun_out/abmc2_cta${c}_$i.err
done; done
