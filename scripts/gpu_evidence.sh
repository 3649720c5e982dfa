#!/bin/bash
# One gpurun call: GPU tests, N=1 bench, ncu launch list, ncu --set full of the top GEMM.
# usage: gpurun -- bash scripts/gpu_evidence.sh TAG
TAG=${1:-r01}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout -s KILL 900 python -m pytest tests -q -m gpu -x --timeout 600 -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout -s KILL 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; tail -1 gpurun_out/${TAG}_bench.json
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
timeout -s KILL 1200 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_launches.log 2>&1
echo "ncu list rc=$?"
timeout -s KILL 1200 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:"gemm_tcgen05" -s 2 -c 1 -o gpurun_out/${TAG}_gemm_full $CMD > gpurun_out/${TAG}_gemm_full.log 2>&1
echo "ncu full gemm rc=$?"
timeout -s KILL 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:"attn_prefix" -c 1 -o gpurun_out/${TAG}_attn_full $CMD > gpurun_out/${TAG}_attn_full.log 2>&1
echo "ncu full attn rc=$?"
