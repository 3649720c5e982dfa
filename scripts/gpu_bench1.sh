timeout -s KILL 300 python bench.py --config c1 2>&1 | tail -5
timeout -s KILL 900 python bench.py --config c3 2>&1 | tail -5
