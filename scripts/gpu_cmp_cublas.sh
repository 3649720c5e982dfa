#!/bin/bash
# ncu --set full of our GEMM (mode given by KRR_GEMM_CTA) and cuBLAS on the MLP-up shape
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for cta in 4 2; do
  KRR_GEMM_CTA=$cta timeout -s KILL 900 ncu --set full --clock-control none -k regex:"gemm_tcgen05|nvjet" -c 2 -o gpurun_out/cmp_cta$cta python scripts/gemm_vs_cublas_ncu.py > gpurun_out/cmp_cta$cta.log 2>&1
  echo "cta=$cta rc=$?"; tail -1 gpurun_out/cmp_cta$cta.log
done
