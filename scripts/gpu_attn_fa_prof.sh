#!/bin/bash
TAG=${1:-fa}
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python scripts/attn_bench.py --pairs 6400 --boost 1 16 --backends mma,tc 2>&1 | tee gpurun_out/${TAG}_micro.txt
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"attn_fa" -s 3 -c 1 -o gpurun_out/${TAG}_attn_full python scripts/attn_bench.py --pairs 1600 --boost 16 --backends tc --reps 2 > gpurun_out/${TAG}_attn_full.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/${TAG}_attn_full.log
