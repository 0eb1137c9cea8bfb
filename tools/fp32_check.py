"""fp32 mode against fp64 on one workload: relative L2 of phi, E and the
energy difference, plus the per-stage times of both."""
import os
import sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np
from paper_2101_07088_b200 import workloads as W
from paper_2101_07088_b200.slab import SlabSolver

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
s, p = W.build(name)
out = {}
for prec in ("fp64", "fp32"):
    solver = SlabSolver(s, p, precision=prec)
    for _ in range(3):
        res = solver.solve(timings=True)
    out[prec] = res
    print(prec, {k: round(v, 3) for k, v in res.diagnostics["timings_ms"].items()})
a, b = out["fp64"], out["fp32"]
rel = lambda x, y: float(np.linalg.norm(x - y) / np.linalg.norm(y))
print("phi rel L2 %.3e  E rel L2 %.3e  U rel %.3e" % (rel(b.phi_bar, a.phi_bar),
      rel(b.E_bar, a.E_bar), abs(b.U - a.U) / abs(a.U)))
