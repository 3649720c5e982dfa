KRR_GEMM_CTA=1 timeout -s KILL 600 python scripts/gemm_bench.py "$@"
KRR_GEMM_CTA=2 timeout -s KILL 600 python scripts/gemm_bench.py "$@"
