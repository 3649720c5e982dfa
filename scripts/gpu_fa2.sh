#!/bin/bash
# fa2 (128-key blocks) vs fa: correctness under KRR_ATTN_TC_KERNEL=fa2, micro-benchmark, C3 A/B
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
KRR_ATTN_TC_KERNEL=fa2 timeout -s KILL 900 python -m pytest tests/test_gpu_kernels.py -k attention -q -x -p no:cacheprovider > gpurun_out/fa2_kern.log 2>&1
echo "fa2 attention tests rc=$?"; grep -E "passed|failed|^FAILED|^E " gpurun_out/fa2_kern.log | tail -6
KRR_ATTN_TC_KERNEL=fa2 timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_depth.py -q -x -p no:cacheprovider > gpurun_out/fa2_par.log 2>&1
echo "fa2 parity tests rc=$?"; grep -E "passed|failed|^FAILED|^E " gpurun_out/fa2_par.log | tail -6
for r in 1 2; do for k in fa fa2; do
  echo "== $k run $r"; KRR_ATTN_TC_KERNEL=$k python scripts/attn_bench.py --pairs 6400 --boost 1 16 --backends tc --reps 30 2>&1 | tail -2
done; done
for r in 1 2; do for k in fa fa2; do
  KRR_ATTN_TC_KERNEL=$k timeout -s KILL 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4 > gpurun_out/fa2_c3_${k}_$r.json 2>/dev/null
  echo -n "c3 $k run $r: "; tail -1 gpurun_out/fa2_c3_${k}_$r.json | python scripts/show.py
done; done
