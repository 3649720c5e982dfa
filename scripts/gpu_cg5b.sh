#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
KRR_GEMM_CTA=6 timeout -s KILL 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_depth.py -q -x -p no:cacheprovider -s > gpurun_out/cg5b_t.log 2>&1
echo "mode6 tests rc=$?"; grep -E "passed|failed|^FAILED|^E |layer" gpurun_out/cg5b_t.log | tail -10
KRR_GEMM_CTA=6 timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tcgen05 -s 1 -c 1 --csv python scripts/gemm_traffic.py 2>/dev/null | grep -E "gpu__time|tensor|per_second" | awk -F'","' '{print "   " $(NF-2) " " $(NF-1) " " $NF}'
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for i in 1 2; do for cta in 4 6; do
  KRR_GEMM_CTA=$cta timeout -s KILL 600 $B > gpurun_out/cg5b_c3_${cta}_$i.json 2>/dev/null
  echo -n "c3 cta=$cta run=$i "; tail -1 gpurun_out/cg5b_c3_${cta}_$i.json | python scripts/show.py
done; done
