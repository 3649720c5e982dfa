set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import paper_2504_02921_b200 as k; print(k.__version__)"
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py -q -k "not TCGEN05 and not tcgen05" --timeout 120 -p no:cacheprovider 2>&1 | tail -30
timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -q -k "tcgen05 or TCGEN05" --timeout 60 -x -p no:cacheprovider 2>&1 | tail -30
