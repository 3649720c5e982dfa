#!/bin/bash
# C5 staging-group size sweep (documents per scoring forward = staging/2).
TAG=${1:-c5stg}
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for qz in int4 int8 ""; do
  for st in 16 32 64; do
    timeout -s KILL 900 python bench.py --config c5 --corpus 200 --steps 5 --warmup 2 --query-lens 16,48,256 --no-cpu-baseline --staging-slots $st ${qz:+--host-quant $qz} > gpurun_out/${TAG}_${qz:-f16}_$st.json 2>/dev/null
    python - "$st" "${qz:-f16}" gpurun_out/${TAG}_${qz:-f16}_$st.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
print(sys.argv[2], "staging", sys.argv[1], " ".join(f"Q{q}:{v['pairs_per_s']:.0f}({v['pairs_per_s']/v['pairs_roofline']:.2f})" for q,v in d["query_len_sweep"].items()))
PY
  done
done
