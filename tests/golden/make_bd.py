"""Brownian-dynamics goldens from the REFERENCE package (build container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_bd.py

Steric pair forces (periodic xy, open z) and wall forces for a dense small
system, steric force / energy curves, and three BD steps (reference Philox
noise, z-bound rejections, xy wrap) driven by fixed forces.  Stored in
bd.npz next to this script.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from slabewald import bd as sb                            # noqa: E402


def main():
    out = {}
    rng = np.random.default_rng(31)
    L, H = 1.0, 0.6
    # jittered lattice: neighbours mostly inside the steric cutoff, no
    # overlaps closer than the capped core
    g = np.arange(16) * (L / 16)
    zg = 0.1 + np.arange(8) * 0.057
    pos = np.stack(np.meshgrid(g, g, zg, indexing="ij"), -1).reshape(-1, 3)
    pos = pos + rng.uniform(-0.012, 0.012, pos.shape)
    pos[:, :2] = np.mod(pos[:, :2], L)
    n = pos.shape[0]
    pos[0] = [0.0, 0.5, 0.3]                 # periodic edge
    pos[1] = [L - 0.01, 0.5, 0.3]            # its neighbour across the edge
    pos[2] = [0.3, 0.3, 0.3]                 # a close pair (capped core)
    pos[3] = [0.3, 0.3, 0.3 + 0.012]
    pos[4, 2] = 0.015                        # near the walls (steric wall force)
    pos[5, 2] = H - 0.012
    for name, st in (("a", sb.StericParams(a=0.02)),
                     ("b", sb.StericParams(a=0.02, U0=2.5, r_m=0.025, p=6)),
                     ("c", sb.StericParams(a=0.015, U0=1.0, r_m=0.0, p=12))):
        out["pos"] = pos
        out["steric_%s" % name] = np.array([st.a, st.U0, st.r_m, st.p])
        out["pair_%s" % name] = sb.steric_pair_forces(pos, st, (L, L, None))
        out["wall_%s" % name] = sb.wall_steric_forces(pos, st, H)
        r = np.linspace(1e-4, 0.1, 257)
        out["r"] = r
        out["force_%s" % name] = sb.steric_force(r, st)
        out["energy_%s" % name] = sb.steric_energy(r, st)
    # three BD steps with fixed forces, z bounds and xy wrap
    cfg = sb.BdConfig(dt=2e-5, steps=3, seed=5, max_disp=0.01)
    pos_bd = pos.copy()
    pos_bd[4:6, 2] = 0.3                     # inside the BD z bounds
    out["bd_pos0"] = pos_bd
    state = sb.make_state(pos_bd, cfg)
    forces = np.random.default_rng(2).standard_normal(pos.shape) * 5.0
    traj = []
    for _ in range(3):
        sb.bd_step(state, forces, cfg, z_bounds=(0.05, H - 0.05), wrap=(L, L, None))
        traj.append(state.positions.copy())
    out["bd_forces"] = forces
    out["bd_traj"] = np.stack(traj)
    out["bd_rejections"] = np.int64(state.rejections)
    np.savez_compressed(os.path.join(HERE, "bd.npz"), **out)
    print("bd.npz", state.rejections, "rejections")


if __name__ == "__main__":
    main()


def bd_loop_golden():
    """Two steps of the cmd_bd loop (cli.py:203-215) on a small C2-box
    electrolyte: forces = q E (solver, need_energy=False) + steric + wall."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    import slabewald as sw
    from paper_2101_07088_b200 import workloads as W
    desc = dict(W.WORKLOADS["c2"])
    geo = sw.SlabGeometry(desc["L"], desc["L"], desc["H"], 1.0, desc["eps_b"], desc["eps_t"])
    pos, q = W.make_inputs(desc, 256)
    system = sw.ChargeSystem(geo, pos, q, desc["g_w"])
    params = sw.plan_grid(geo, desc["g_w"], desc["delta"], Nxy=desc["Nxy"])
    solver = sw.SlabSolver(system, params)
    st = sb.StericParams(a=0.01)
    cfg = sb.BdConfig(dt=1e-6, steps=2, seed=3, max_disp=st.a)
    margin = params.n_sigma * system.g_w
    state = sb.make_state(system.positions, cfg)
    traj = []
    for _ in range(2):
        res = solver.solve(positions=state.positions, need_energy=False)
        f = res.forces + sb.steric_pair_forces(state.positions, st, (geo.Lx, geo.Ly, None)) \
            + sb.wall_steric_forces(state.positions, st, geo.H)
        sb.bd_step(state, f, cfg, z_bounds=(margin, geo.H - margin), wrap=(geo.Lx, geo.Ly, None))
        traj.append(state.positions.copy())
    np.savez_compressed(os.path.join(HERE, "bd_loop.npz"), traj=np.stack(traj),
                        rejections=np.int64(state.rejections))
    print("bd_loop.npz", state.rejections, "rejections")


if __name__ == "__main__" and "--loop" in sys.argv:
    bd_loop_golden()
