timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -p no:cacheprovider 2>&1 | tail -40
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
