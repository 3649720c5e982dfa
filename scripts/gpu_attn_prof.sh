#!/bin/bash
# attention kernel tests, C3 bench, ncu full capture of the tcgen05 attention kernel.
TAG=${1:-attn}
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --latency-reps 5 --full-pairs 16 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; python scripts/show.py gpurun_out/${TAG}_bench.json 2>/dev/null || tail -c 600 gpurun_out/${TAG}_bench.json
CMD="python bench.py --queries 8 --cands 100 --corpus 100 --steps 1 --warmup 1 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
timeout -s KILL 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:"attn_(tc|pp)" -c 1 -o gpurun_out/${TAG}_attn_full $CMD > gpurun_out/${TAG}_attn_full.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/${TAG}_attn_full.log
