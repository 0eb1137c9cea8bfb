"""One warm C4 solve in fp32 mode (ncu captures)."""
import os
import sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2101_07088_b200 import workloads as W
from paper_2101_07088_b200.slab import SlabSolver

s, p = W.build(sys.argv[1] if len(sys.argv) > 1 else "c4")
solver = SlabSolver(s, p, precision="fp32")
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    res = solver.solve(timings=True)
print(res.diagnostics["timings_ms"])
