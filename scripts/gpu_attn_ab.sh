#!/bin/bash
# A/B of the attention kernel: tests, micro-benchmark (boost 1/8/16), C3 bench
TAG=${1:-ab}
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_depth.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^E " gpurun_out/${TAG}_pytest.log | tail -8
python scripts/attn_bench.py --pairs 6400 --boost 1 8 16 --backends tc 2>&1 | tee gpurun_out/${TAG}_micro.txt
for i in 1 2; do
timeout -s KILL 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4 > gpurun_out/${TAG}_c3_$i.json 2>/dev/null
echo -n "c3 "; tail -1 gpurun_out/${TAG}_c3_$i.json | python scripts/show.py
done
