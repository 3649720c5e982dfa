#!/bin/bash
# C3 step A/B between variant libraries (KRR_LIB), alternating; args: variant names (default = main lib)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
P=$PWD/paper_2504_02921_b200
timeout -s KILL 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/libab_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^E " gpurun_out/libab_pytest.log | tail -4
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for i in 1 2 3; do for v in "$@"; do
  lib=$P/_krr_$v.so; [ "$v" = default ] && lib=$P/_kvrerank_b200.so
  KRR_LIB=$lib timeout -s KILL 600 $B > gpurun_out/libab_${v}_$i.json 2>/dev/null
  echo -n "$v run=$i "; tail -1 gpurun_out/libab_${v}_$i.json | python scripts/show.py
done; done
