#!/bin/bash
# wave-model N-tile width: correctness, GEMM micro at the latency batch, p50 latency A/B
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/wave_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^E " gpurun_out/wave_pytest.log | tail -8
for nn in 1 0; do
  echo "== KRR_GEMM_NARROW=$nn gemm M=4800"
  KRR_GEMM_NARROW=$nn timeout -s KILL 300 python scripts/gemm_bench.py --m 4800 --reps 50 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    l = l.strip()
    if l.startswith('{'):
        d = json.loads(l)
        print('  ', {k: (v['ms'], v['tflops']) for k, v in d.items() if isinstance(v, dict) and 'ms' in v and 'cublas' not in k})
"
done
for r in 1 2; do for nn in 1 0; do
  KRR_GEMM_NARROW=$nn timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --latency-reps 20 --full-pairs 4 > gpurun_out/wave_c3_${nn}_$r.json 2>/dev/null
  echo -n "c3 narrow=$nn run $r: "; tail -1 gpurun_out/wave_c3_${nn}_$r.json | python scripts/show.py
  KRR_GEMM_NARROW=$nn timeout -s KILL 900 python bench.py --config c2 --steps 20 --warmup 3 --no-cpu-baseline --latency-reps 20 > gpurun_out/wave_c2_${nn}_$r.json 2>/dev/null
  echo -n "c2 narrow=$nn run $r: "; tail -1 gpurun_out/wave_c2_${nn}_$r.json | python scripts/show.py
done; done
