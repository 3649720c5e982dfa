#!/bin/bash
# A/B of GEMM tile shape (KRR_GEMM_CTA) and L2 rasterisation (KRR_GEMM_GROUP_M) on the full C3 bench.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
for cfg in "1 16" "1 64" "1 128" "2 8" "2 32"; do
  set -- $cfg
  KRR_GEMM_CTA=$1 KRR_GEMM_GROUP_M=$2 timeout -s KILL 600 $B > gpurun_out/knob_cta$1_gm$2.json 2>&1
  python - "$1" "$2" <<'PY'
import json,sys
l=open(f"gpurun_out/knob_cta{sys.argv[1]}_gm{sys.argv[2]}.json").read().strip().splitlines()[-1]
try:
  d=json.loads(l); r=d["roofline"]
  print("cta",sys.argv[1],"gm",sys.argv[2],"pairs/s %.1f gemmTF %.1f share %.3f attn %.3f clk %s"%(d["value"],r["achieved"],r["gemm_share_of_step"],r["attn_share_of_step"],d["clocks"]))
except Exception as e: print("FAIL",sys.argv[1:],l[-300:])
PY
done
