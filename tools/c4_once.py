"""One warm C4 solve (for ncu launch lists / captures)."""
import os
import sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2101_07088_b200 import workloads as W
from paper_2101_07088_b200.slab import SlabSolver

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
s, p = W.build(name, N=int(sys.argv[3]) if len(sys.argv) > 3 else None)
solver = SlabSolver(s, p)
for _ in range(reps):
    res = solver.solve(timings=True)
print(name, res.diagnostics["timings_ms"], "U", res.U, "launches",
      res.diagnostics["n_launches"])
