#!/bin/bash
# correctness of a variant library (attention tests) + micro + C3 A/B vs the default
V=$1
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
P=$PWD/paper_2504_02921_b200
KRR_LIB=$P/_krr_$V.so timeout -s KILL 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/vt_$V.log 2>&1
echo "$V tests rc=$?"; grep -E "passed|failed|^FAILED|^E " gpurun_out/vt_$V.log | tail -4
bash scripts/gpu_attn_variants.sh default $V
for r in 1 2; do for v in default $V; do
  lib=$P/_krr_$v.so; [ "$v" = default ] && lib=$P/_kvrerank_b200.so
  KRR_LIB=$lib timeout -s KILL 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4 > gpurun_out/vt_c3_${v}_$r.json 2>/dev/null
  echo -n "c3 $v run $r: "; tail -1 gpurun_out/vt_c3_${v}_$r.json | python scripts/show.py
done; done
