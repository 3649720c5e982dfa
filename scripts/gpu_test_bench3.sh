#!/bin/bash
# GPU tests then a short C3 bench.  usage: gpurun -- bash scripts/gpu_test_bench3.sh TAG [bench args]
TAG=${1:-iter}; shift
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider -x > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -25 gpurun_out/${TAG}_pytest.log | grep -E "passed|failed|Error|error|assert" | head -20
timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --latency-reps 5 --full-pairs 16 "$@" > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; tail -c 1500 gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
