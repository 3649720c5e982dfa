#!/bin/bash
TAG=${1:-c5}
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for qz in "" int8 int4; do
  timeout -s KILL 900 python bench.py --config c5 --steps 3 --warmup 2 --query-lens 16,48,256 --no-cpu-baseline ${qz:+--host-quant $qz} > gpurun_out/${TAG}_c5_${qz:-f16}.json 2> gpurun_out/${TAG}_c5_${qz:-f16}.err
  echo -n "c5 ${qz:-f16} rc=$? "; python - "$TAG" "${qz:-f16}" <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/{sys.argv[1]}_c5_{sys.argv[2]}.json").read().strip().splitlines()[-1])
print({q:(round(v["pairs_per_s"],1), round(v["h2d_gbs"],1), round(v["pairs_roofline"],1)) for q,v in d["query_len_sweep"].items()})
PY
done
