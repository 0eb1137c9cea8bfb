"""Reference goldens at the north-star grid and density.

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_c4.py

Runs the REFERENCE package ``slabewald`` on
  * ``c4n64k``: the C4 box and grid (L=2, H=1, 256 x 256 x 258, eps 0.05 at
    both walls, delta 1e-4) with N = 65536 of the C4 workload's charges;
  * ``c4d``: C4 density and spacing in a 0.5 x 0.5 box (64 x 64 x 258,
    N = 65536, ~575 near pairs per charge).
Stores phi, E, U and the diagnostics of ``SlabSolver.solve()`` and, for
``c4d``, the near-field pair SET of ``NearField._pairs`` (slab.py:133-148)
as per-target counts and order-independent hashes (tests/_golden.py
``pair_hash``) -- 37.7 M pairs do not fit in a fixture.  Output:
tests/golden/c4.npz.
"""
import os
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

import slabewald as sw                                   # noqa: E402
from slabewald import slab as sw_slab                    # noqa: E402

from make_golden import ref_problem, outputs             # noqa: E402
from _golden import pair_hash                            # noqa: E402


def main():
    warnings.simplefilter("ignore")
    out = {}
    for case, name in (("c4n64k", "c4"), ("c4d", "c4d")):
        s, p = ref_problem(name, N=65536)
        print(case, "grid %dx%dx%d xi %.4f r_cut %.5f" % (p.Nx, p.Ny, p.Nz, p.xi, p.r_cut),
              flush=True)
        t = time.time()
        res = sw.SlabSolver(s, p).solve()
        print("   solve %.1fs" % (time.time() - t), flush=True)
        for k, v in outputs(res).items():
            out["%s__%s" % (case, k)] = v
        if case == "c4d":
            nf = sw_slab.NearField(s.positions, s.charges, s.geometry, p)
            e, src, _d, _r = nf._pairs(s.positions, p.r_cut)
            cnt, h = pair_hash(e, src, s.positions.shape[0])
            out[case + "__pair_count"] = cnt.astype(np.int32)
            out[case + "__pair_hash"] = h
            out[case + "__n_pairs"] = np.int64(e.size)
            print("   pairs %d (%.1f per charge)" % (e.size, e.size / cnt.size), flush=True)
    np.savez_compressed(os.path.join(HERE, "c4.npz"), **out)
    print("c4.npz")


if __name__ == "__main__":
    main()
