#!/bin/bash
# attention A/B: correctness of the default build, then variant micro-benchmarks and C3
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_depth.py -q -x -p no:cacheprovider > gpurun_out/ab2_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^E " gpurun_out/ab2_pytest.log | tail -8
bash scripts/gpu_attn_variants.sh "$@"
P=$PWD/paper_2504_02921_b200
for r in 1 2; do for v in "$@"; do
  lib=$P/_krr_$v.so; [ "$v" = default ] && lib=$P/_kvrerank_b200.so
  KRR_LIB=$lib timeout -s KILL 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4 > gpurun_out/ab2_c3_${v}_$r.json 2>/dev/null
  echo -n "c3 $v run $r: "; tail -1 gpurun_out/ab2_c3_${v}_$r.json | python scripts/show.py
done; done
