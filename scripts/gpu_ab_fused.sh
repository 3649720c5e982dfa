#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -x > gpurun_out/fused_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^E " gpurun_out/fused_pytest.log | tail -8
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for i in 1 2; do for f in 1 0; do
  KRR_FUSED_NORM=$f timeout -s KILL 600 $B > gpurun_out/abf_${f}_$i.json 2>gpurun_out/abf_${f}_$i.err
  echo -n "fused=$f run=$i "; tail -1 gpurun_out/abf_${f}_$i.json | python scripts/show.py; tail -1 gpurun_out/abf_${f}_$i.err
done; done
