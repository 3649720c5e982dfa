#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_store.py tests/test_gpu_depth.py -q -x -p no:cacheprovider > gpurun_out/c5t_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^E " gpurun_out/c5t_pytest.log | tail -8
timeout -s KILL 600 python scripts/c5_trace.py 16 16 2>&1 | grep -v "^  g"
timeout -s KILL 600 python scripts/c5_trace.py 16 32 2>&1 | tail -30
timeout -s KILL 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4 > gpurun_out/c5t_c3.json 2>/dev/null
echo -n "c3 "; tail -1 gpurun_out/c5t_c3.json | python scripts/show.py
timeout -s KILL 600 python bench.py --config c2 --steps 20 --warmup 3 --no-cpu-baseline --latency-reps 15 > gpurun_out/c5t_c2.json 2>/dev/null
echo -n "c2 "; tail -1 gpurun_out/c5t_c2.json | python scripts/show.py
