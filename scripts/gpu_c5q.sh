#!/bin/bash
TAG=${1:-c5q}
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_store.py -q --timeout 600 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^E " gpurun_out/${TAG}_pytest.log | tail -8
timeout -s KILL 300 python scripts/c5_probe.py 2>&1 | tail -4
for qz in "" int8 int4; do
timeout -s KILL 900 python bench.py --config c5 --steps 3 --warmup 1 --query-lens 16,48,256 ${qz:+--host-quant $qz} > gpurun_out/${TAG}_c5_${qz:-f16}.json 2> gpurun_out/${TAG}_c5_${qz:-f16}.err
echo "c5 $qz rc=$?"; python - "$TAG" "${qz:-f16}" <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/{sys.argv[1]}_c5_{sys.argv[2]}.json").read().strip().splitlines()[-1])
print(sys.argv[2], "h2d_peak %.1f"%d["h2d_peak_gbs"], {q:(round(v["pairs_per_s"],1), round(v["h2d_gbs"],1), round(v["reuse_over_full"],2)) for q,v in d["query_len_sweep"].items()})
PY
done
