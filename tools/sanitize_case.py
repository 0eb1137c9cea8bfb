"""Small solves for compute-sanitizer runs (memcheck / racecheck /
synccheck): C2 (N=2048, fp64, fp32 mode, pair-set record, graph replay)
and a C3-box case at N=48000 so the large-N near-field list path runs.

    compute-sanitizer --tool memcheck python tools/sanitize_case.py [small]
"""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2101_07088_b200 import workloads as W          # noqa: E402
from paper_2101_07088_b200.slab import SlabSolver        # noqa: E402

small = len(sys.argv) > 1 and sys.argv[1] == "small"
s, p = W.build("c2", N=512 if small else 2048)
for prec in ("fp64", "fp32"):
    sv = SlabSolver(s, p, precision=prec)
    r = sv.solve(record_pairs=True)
    sv.pair_set()
    assert np.all(np.isfinite(r.phi_bar))
    sv.close()
if not small:
    s3, p3 = W.build("c3", N=48000)
    sv = SlabSolver(s3, p3)
    r = sv.solve()
    assert np.all(np.isfinite(r.E_bar))
    sv.close()
print("ok")
