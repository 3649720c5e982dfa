# usage: bash scripts/gpu_test_bench.sh [bench args...]
timeout -s KILL 900 python -m pytest tests -q -m gpu --timeout 300 -x -p no:cacheprovider 2>&1 | tail -15
timeout -s KILL 900 python bench.py --no-cpu-baseline "$@" 2>&1 | tail -3
