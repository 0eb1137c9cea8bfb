import os, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2101_07088_b200 import _lib
_lib.LIB_PATH = os.path.join(REPO, "tools", "libse_stats.so")
from paper_2101_07088_b200 import workloads as W
from paper_2101_07088_b200.slab import SlabSolver
s, p = W.build("c4")
solver = SlabSolver(s, p)
solver.solve()
