"""Triply periodic twin goldens from the REFERENCE package (build container):

    python tests/golden/make_tp.py

solve_triply_periodic on two seeded grids (even and odd sizes, with and
without the field), TriplyPeriodicSolver.forces and the fully periodic
steric forces on the g2 experiment's electrolyte (validate.py:218-246, fewer
ions), and two steps of that experiment's BD loop.  Stored in tp.npz next to
this script.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import slabewald as sw                                     # noqa: E402
from slabewald import bd as sb                             # noqa: E402
from slabewald import validate as sv                       # noqa: E402


def main():
    out = {}
    rng = np.random.default_rng(17)
    for tag, shape, box in (("a", (12, 10, 9), (1.0, 0.8, 0.9)),
                            ("b", (16, 16, 16), (2.0, 2.0, 2.0))):
        rho = rng.standard_normal(shape)
        phi, e = sw.solve_triply_periodic(rho, 0.7, *box, with_field=True)
        out["rho_" + tag] = rho
        out["box_" + tag] = np.array(box)
        out["phi_" + tag] = phi
        out["e_" + tag] = e
        out["phi_only_" + tag] = sw.solve_triply_periodic(rho, 0.7, *box)
    # the g2 electrolyte (validate.py:218-246) with 400 ions
    n_ions, molar = 400, 0.05
    dens = sv.electrolyte_number_density(molar)
    lam_b = sv.BJERRUM_M / sv.ION_RADIUS_M
    eps = 1.0 / (4.0 * np.pi * lam_b)
    box = (n_ions / dens) ** (1.0 / 3.0)
    steric = sb.StericParams(a=1.0, U0=0.2233, r_m=1.0, p=2)
    solver = sb.TriplyPeriodicSolver((box, box, box), 32, 0.25, eps, delta=5e-4)
    pos = rng.uniform(0.0, box, (n_ions, 3))
    charges = np.tile([1.0, -1.0], n_ions // 2)
    out.update(g2_box=np.float64(box), g2_eps=np.float64(eps), g2_pos=pos,
               g2_q=charges, g2_forces=solver.forces(pos, charges),
               g2_steric=sb.steric_pair_forces(pos, steric, (box, box, box)),
               g2_rcut=np.float64(solver.r_cut), g2_n=np.array(solver.grid.n))
    cfg = sb.BdConfig(dt=5e-3, steps=2, seed=42, max_disp=1.0)
    state = sb.make_state(pos, cfg)
    traj = []
    for _ in range(2):
        f = solver.forces(state.positions, charges) \
            + sb.steric_pair_forces(state.positions, steric, (box, box, box))
        sb.bd_step(state, f, cfg, wrap=(box, box, box))
        traj.append(state.positions.copy())
    out["g2_traj"] = np.stack(traj)
    np.savez_compressed(os.path.join(HERE, "tp.npz"), **out)
    print("tp.npz box %.3f r_cut %.3f grid %s" % (box, solver.r_cut, solver.grid.n))


if __name__ == "__main__":
    main()
