#!/bin/bash
# mode 6 (Cfg<5>: 256 rows per CTA, two MMAs share a B stage): correctness, GEMM micro, C3 A/B
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
KRR_GEMM_CTA=6 timeout -s KILL 900 python -m pytest tests/test_gpu_kernels.py -k gemm -q -x -p no:cacheprovider > gpurun_out/cg5_kern.log 2>&1
echo "mode6 gemm tests rc=$?"; grep -E "passed|failed|^FAILED|^E " gpurun_out/cg5_kern.log | tail -5
KRR_GEMM_CTA=6 timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_depth.py -q -x -p no:cacheprovider > gpurun_out/cg5_par.log 2>&1
echo "mode6 parity rc=$?"; grep -E "passed|failed|^FAILED|^E " gpurun_out/cg5_par.log | tail -5
for cta in 4 6; do
  echo "== gemm_bench CTA=$cta"
  KRR_GEMM_CTA=$cta timeout -s KILL 600 python scripts/gemm_bench.py --m 65536 --reps 200 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    l = l.strip()
    if l.startswith('{'):
        d = json.loads(l)
        for k, v in d.items():
            if isinstance(v, dict) and 'ms' in v and 'cublas' not in k:
                print(f\"   {k:10s} {v['ms']:.3f} ms {v['tflops']:7.1f} TF/s {v['sm_mhz']:.0f} MHz {v['watts']:.0f} W\")
"
done
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for i in 1 2; do for cta in 4 6; do
  KRR_GEMM_CTA=$cta timeout -s KILL 600 $B > gpurun_out/cg5_c3_${cta}_$i.json 2>/dev/null
  echo -n "c3 cta=$cta run=$i "; tail -1 gpurun_out/cg5_c3_${cta}_$i.json | python scripts/show.py
done; done
