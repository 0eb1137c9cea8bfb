"""Free-space slab agreement golden (the reference's validate suite
`freespace`, validate.py:110-132; PAPER Table 2: 9.755e-6):

    python tests/golden/make_freespace.py

Stores the 400-image open-slab oracle field, the reference solver's E_bar at
L = 28 and 32 and its extrapolated error in freespace.npz next to this
script.
"""

import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import slabewald as sw                                    # noqa: E402
from slabewald import validate as v                       # noqa: E402
from slabewald.reference import (free_space_slab_reference,  # noqa: E402
                                 richardson_infinite_box)


def main():
    g_w, H = 1e-2, 2.0
    geo = sw.SlabGeometry(1.0, 1.0, H, eps=1.0, eps_b=0.5, eps_t=0.2)
    phi_f, e_f = free_space_slab_reference(v.FREESPACE_CHARGES, v.FREESPACE_Q, g_w, geo,
                                           n_levels=100)
    out = {"charges": v.FREESPACE_CHARGES, "q": v.FREESPACE_Q, "e_f": e_f}
    fields = {}
    for L in (28.0, 32.0):
        g = sw.SlabGeometry(L, L, H, eps=1.0, eps_b=0.5, eps_t=0.2)
        pos = v.FREESPACE_CHARGES.copy()
        pos[:, :2] += 0.5 * L
        system = sw.ChargeSystem(g, pos, v.FREESPACE_Q, g_w)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            params = sw.plan_grid(g, g_w, 1e-4, xi=3.0177, h_min=0.01, strict=False)
        fields[L] = sw.SlabSolver(system, params).solve().E_bar
        out["E_L%d" % int(L)] = fields[L]
    e_inf = richardson_infinite_box(fields[28.0], 28.0, fields[32.0], 32.0)
    out["err"] = np.float64(np.max(np.abs(e_inf - e_f)) / np.mean(np.linalg.norm(e_f, axis=1)))
    np.savez_compressed(os.path.join(HERE, "freespace.npz"), **out)
    print("freespace err", out["err"])


if __name__ == "__main__":
    main()
