#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/var_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^E " gpurun_out/var_pytest.log | tail -12
timeout -s KILL 900 python bench.py --config c3r --steps 4 --warmup 3 --no-cpu-baseline --latency-reps 5 --full-pairs 4 > gpurun_out/var_c3r.json 2> gpurun_out/var_c3r.err
echo -n "c3r rc=$? "; tail -1 gpurun_out/var_c3r.json | python scripts/show.py; tail -2 gpurun_out/var_c3r.err
