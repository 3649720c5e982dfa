#!/bin/bash
# compute-sanitizer memcheck / racecheck over the kernel, grouped-attention, fused-dequant,
# parity and store tests.  usage: gpurun -- bash scripts/gpu_sanitizer.sh TAG
TAG=${1:-san}
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
run() {  # name tool pytest-args...
  local name=$1 tool=$2; shift 2
  timeout -s KILL 1500 compute-sanitizer --tool $tool --target-processes all python -m pytest "$@" -q -m gpu -p no:cacheprovider > gpurun_out/${TAG}_$name.log 2>&1
  echo "$name ($tool) rc=$?: $(grep -E 'passed|failed' gpurun_out/${TAG}_$name.log | tail -1) | $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/${TAG}_$name.log | sort | uniq -c | tr '\n' ' ')"
}
run mem_kernels memcheck tests/test_gpu_kernels.py -k "attention and 128 or attention and 256 or quant or gemm_store or gated or pair_geometry"
run mem_e2e memcheck tests/test_gpu_grouped.py tests/test_gpu_parity.py tests/test_gpu_store.py
run race_attn racecheck tests/test_gpu_kernels.py -k "quant_prefix and 512 or attention and 128 and 512 and F16 or attention and 256 and 512"
run race_grouped racecheck tests/test_gpu_grouped.py -k "f16"
