#!/bin/bash
# Final committed tree: GPU suite, smoke, default C3 line, C2 line (graph-timed step).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TAG=${1:-r02g}
timeout -s KILL 1500 python -m pytest tests -q -m gpu --timeout 1200 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^ERROR" gpurun_out/${TAG}_pytest.log | tail -6
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout -s KILL 1500 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo -n "bench rc=$? "; python scripts/show.py gpurun_out/${TAG}_bench.json
timeout -s KILL 900 python bench.py --config c2 --steps 20 --warmup 3 --latency-reps 15 > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.err
echo -n "c2 rc=$? "; python scripts/show.py gpurun_out/${TAG}_c2.json
