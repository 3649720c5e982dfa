#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_depth.py -q -x -p no:cacheprovider > gpurun_out/narrow_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^E " gpurun_out/narrow_pytest.log | tail -8
for i in 1 2; do for nn in 0 2560; do
  KRR_GEMM_NARROW=$nn timeout -s KILL 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline --latency-reps 15 > gpurun_out/abn_c2_${nn}_$i.json 2>/dev/null
  echo -n "c2 narrow=$nn run=$i "; tail -1 gpurun_out/abn_c2_${nn}_$i.json | python scripts/show.py
done; done
for nn in 0 2560; do
  KRR_GEMM_NARROW=$nn timeout -s KILL 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4 > gpurun_out/abn_c3_${nn}.json 2>/dev/null
  echo -n "c3 narrow=$nn "; tail -1 gpurun_out/abn_c3_${nn}.json | python scripts/show.py
done
