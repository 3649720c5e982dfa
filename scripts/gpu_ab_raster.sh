#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -1
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for i in 1 2; do for r in auto m; do
  KRR_GEMM_RASTER=$r timeout -s KILL 600 $B > gpurun_out/abr_${r}_$i.json 2>gpurun_out/abr_${r}_$i.err
  echo -n "raster=$r run=$i "; tail -1 gpurun_out/abr_${r}_$i.json | python scripts/show.py; tail -1 gpurun_out/abr_${r}_$i.err
done; done
