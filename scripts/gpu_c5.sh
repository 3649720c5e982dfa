#!/bin/bash
TAG=${1:-c5}
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
free -g | head -2; nproc
timeout -s KILL 900 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED" gpurun_out/${TAG}_pytest.log | tail -5
timeout -s KILL 900 python bench.py --config c5 --steps 2 --warmup 1 --query-lens 16,48,128,256 > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err
echo "c5 rc=$?"; tail -c 2500 gpurun_out/${TAG}_c5.json; tail -3 gpurun_out/${TAG}_c5.err
timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --latency-reps 5 --full-pairs 16 --no-cpu-baseline > gpurun_out/${TAG}_c3.json 2> gpurun_out/${TAG}_c3.err
echo "c3 rc=$?"; python scripts/show.py gpurun_out/${TAG}_c3.json
