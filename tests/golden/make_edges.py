"""Edge-case goldens from the REFERENCE package (run in the build container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_edges.py

Small systems on the C2 box exercising the boundaries of the path:
coincident charges (r = 0 between distinct charges), charges exactly on grid
nodes, a pair at exactly the cutoff distance, charges on the walls (their
images coincide with them), charges on the periodic edge (x = 0, L - ulp,
L), a single charge and an empty system.  Outputs, or the exception class
the reference raises, are stored in ``edges.npz``.
"""

import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.dirname(HERE))               # tests/ (_edge_cases)
sys.path.insert(0, "/root/reference/pkg/src")

import slabewald as sw                                   # noqa: E402

import _edge_cases as EC                                  # noqa: E402


def main():
    warnings.simplefilter("ignore")
    out = {}
    for name in EC.CASES:
        geo_args, pos, q, g_w, delta, nxy = EC.build(name)
        geo = sw.SlabGeometry(*geo_args)
        p = sw.plan_grid(geo, g_w, delta, Nxy=nxy)
        try:
            s = sw.ChargeSystem(geo, pos, q, g_w)
            res = sw.SlabSolver(s, p).solve()
            out[name + "__phi"] = res.phi_bar
            out[name + "__E"] = res.E_bar
            out[name + "__U"] = np.float64(res.U)
            out[name + "__B_i"] = np.float64(res.diagnostics["B_i"])
            npairs = 0
            if len(q):
                nf = sw.slab.NearField(pos, q, geo, p)
                npairs = len(nf._pairs(pos, p.r_cut)[0])
            out[name + "__npairs"] = np.int64(npairs)
            print(name, "ok", npairs, "pairs", "U", res.U)
        except Exception as exc:                         # noqa: BLE001
            out[name + "__error"] = np.array(type(exc).__name__)
            print(name, "raises", type(exc).__name__, exc)
    np.savez_compressed(os.path.join(HERE, "edges.npz"), **out)


if __name__ == "__main__":
    main()
