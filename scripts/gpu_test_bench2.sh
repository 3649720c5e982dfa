timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 60 -p no:cacheprovider 2>&1 | tail -5 || exit 1
timeout -s KILL 600 python -m pytest tests -q -m gpu --timeout 300 -x -p no:cacheprovider 2>&1 | tail -5
timeout -s KILL 900 python bench.py --no-cpu-baseline "$@" 2>&1 | tail -1
KRR_GEMM_CTA=1 timeout -s KILL 900 python bench.py --no-cpu-baseline "$@" 2>&1 | tail -1
