#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python scripts/attn_bench.py --boost 1 8 16 --backends mma,tc 2>&1 | tee gpurun_out/attn_micro.txt
echo "--- v1 one-tile kernel"; KRR_ATTN_TC_V1=1 python scripts/attn_bench.py --boost 1 16 --backends tc 2>&1 | tee -a gpurun_out/attn_micro.txt
echo "--- pp without rescale"; KRR_LIB=$PWD/paper_2504_02921_b200/_krr_norescale.so python scripts/attn_bench.py --boost 1 16 --backends tc 2>&1 | tee -a gpurun_out/attn_micro.txt
