#!/bin/bash
# Final tree: C4 capacity line and the C5 INT4 host tier at the RAM cap.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TAG=${1:-r02g}
timeout -s KILL 900 python bench.py --config c4 --steps 3 --warmup 3 --latency-reps 5 --no-cpu-baseline > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err
echo -n "c4 rc=$? "; python scripts/show.py gpurun_out/${TAG}_c4.json
timeout -s KILL 900 python bench.py --config c5 --corpus -1 --steps 5 --warmup 3 --query-lens 16,48,256 --no-cpu-baseline --host-quant int4 > gpurun_out/${TAG}_c5_int4.json 2> gpurun_out/${TAG}_c5_int4.err
echo "c5 int4 rc=$?"; tail -c 400 gpurun_out/${TAG}_c5_int4.json
