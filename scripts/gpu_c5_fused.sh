#!/bin/bash
# C5 host tier (f16 / int8 / int4) sweep over query length; quantised tiers use the
# in-attention dequant.  usage: gpurun -- bash scripts/gpu_c5_fused.sh TAG [extra bench args]
TAG=${1:-c5}; shift
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
free -g | head -2
for qz in "" int8 int4; do
  timeout -s KILL 900 python bench.py --config c5 --steps 3 --warmup 2 --query-lens 16,48,256 --no-cpu-baseline ${qz:+--host-quant $qz} "$@" > gpurun_out/${TAG}_c5_${qz:-f16}.json 2> gpurun_out/${TAG}_c5_${qz:-f16}.err
  echo "c5 ${qz:-f16} rc=$?"; tail -2 gpurun_out/${TAG}_c5_${qz:-f16}.err
  python - gpurun_out/${TAG}_c5_${qz:-f16}.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(d["config"]["workload"])
for q, v in d["query_len_sweep"].items():
    print(f"  Q={q}: {v['pairs_per_s']:.1f} pairs/s  h2d {v['h2d_gbs']:.1f} GB/s ({v['h2d_frac_of_peak']:.2f} of peak)  roof {v['pairs_roofline']:.1f}  full {v['full_recompute_pairs_per_s']:.1f}")
PY
done
