#!/bin/bash
TAG=${1:-attnq}
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py -q -k attention --timeout 300 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
CMD="python bench.py --queries 8 --cands 100 --corpus 100 --steps 1 --warmup 1 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
timeout -s KILL 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:"attn_(tc|pp)" -c 1 -o gpurun_out/${TAG}_attn_full $CMD > gpurun_out/${TAG}_attn_full.log 2>&1
echo "ncu rc=$?"; python scripts/ncu_summary.py gpurun_out/${TAG}_attn_full.ncu-rep 2>/dev/null | head -3
