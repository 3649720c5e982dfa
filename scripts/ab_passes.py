"""A/B helper: run bench.py with the scoring/prefill pass split either balanced
(the engine default) or greedy (the round-2 split: full passes plus a tail).
usage: python scripts/ab_passes.py balanced|greedy [bench args...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_02921_b200 import engine
mode = sys.argv.pop(1)
if mode == "greedy":
    engine._balanced_step = lambda n, cap: cap
import bench
sys.argv[0] = bench.__file__
bench.main()
