"""Generate the golden fixtures by RUNNING THE REFERENCE package.

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports ``slabewald`` 0.1.0 from ``/root/reference/pkg/src``, rebuilds
the workloads of ``paper_2101_07088_b200.workloads`` with the REFERENCE's
own classes and planner, and stores its outputs (and, for two small cases,
per-stage intermediates) as ``.npz`` / ``.json`` next to this script.  The
reference ships no fixtures of its own, so these are
the parity anchors for both the oracle and the GPU path.
"""

import json
import os
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import slabewald as sw                                   # noqa: E402
from slabewald import slab as sw_slab                    # noqa: E402
from slabewald import bvp as sw_bvp                      # noqa: E402
from slabewald import chebyshev as sw_cheb               # noqa: E402
from slabewald import reference as sw_ref                # noqa: E402
from slabewald.params import EwaldParams                 # noqa: E402

from paper_2101_07088_b200 import workloads as W         # noqa: E402


def ref_problem(name, N=None, surface=None, **override):
    """Reference (system, params) for workload ``name``."""
    desc = dict(W.WORKLOADS[name])
    desc.update(override)
    geo = sw.SlabGeometry(desc["L"], desc["L"], desc["H"], 1.0,
                          desc["eps_b"], desc["eps_t"])
    pos, q = W.make_inputs(desc, N)
    system = sw.ChargeSystem(geo, pos, q, desc["g_w"], surface)
    if "hand" in desc:
        hp = W.hand_params(desc)
        params = EwaldParams(**{k: getattr(hp, k) for k in (
            "xi", "g_w", "g_t", "delta", "n_g", "n_sigma", "h_xy", "H_E",
            "r_nf", "r_cut", "k_max", "Nx", "Ny", "Nz", "z0", "z1",
            "h_min")})
    else:
        params = sw.plan_grid(geo, desc["g_w"], desc["delta"],
                              Nxy=desc["Nxy"])
    return system, params


def outputs(res):
    d = res.diagnostics
    k0 = d["k0"]
    return dict(phi=res.phi_bar, E=res.E_bar, U=np.float64(res.U),
                ai1=np.float64(d["ai1"]), ai2=np.float64(d["ai2"]),
                disc=np.float64(d["ai_discrepancy"]),
                B_i=np.float64(d["B_i"]), A_i=np.float64(k0.A_i))


def run_solve(system, params, refine=1, **kw):
    t = time.time()
    res = sw.SlabSolver(system, params, refine=refine).solve(**kw)
    print("   solve %.2fs" % (time.time() - t))
    return res


def capture_stages(system, params):
    """Re-run the reference solve with its stage functions wrapped, keeping
    the intermediates (spread grids, psi coefficients, mismatches,
    corrections, field stack, near/far splits)."""
    solver = sw.SlabSolver(system, params)
    cap = {}
    spreads = []
    orig_spread = solver._spread

    def spread(pos, q):
        out = orig_spread(pos, q)
        spreads.append(out)
        return out
    solver._spread = spread
    orig_dtn = solver.dtn.solve

    def dtn(rho, refine=1):
        out = orig_dtn(rho, refine=refine)
        cap["psi"] = out
        return out
    solver.dtn.solve = dtn
    orig_apply = solver.correction.apply

    def apply(m):
        cap["mism"] = m
        out = orig_apply(m)
        cap["corr"], cap["dcorr"] = out
        return out
    solver.correction.apply = apply
    orig_interp = solver.grid.interpolate

    def interp(fields, pos, *a):
        out = orig_interp(fields, pos, *a)
        if np.asarray(fields).ndim == 4:
            cap["fields"] = np.asarray(fields)
            cap["far"] = out
        return out
    solver.grid.interpolate = interp
    res = solver.solve()
    part = sw.build_partition(system.positions, system.charges,
                              system.geometry, params)
    nf = sw_slab.NearField(system.positions, system.charges,
                           system.geometry, params)
    eidx, sidx, d, r = nf._pairs(system.positions, params.r_cut)
    out = outputs(res)
    out.update(rho_over=spreads[0], rho_far=spreads[1],
               psi_o=cap["psi"][0], psi_i=cap["psi"][1],
               m_phi_b=cap["mism"].phi_b, m_e_b=cap["mism"].e_b,
               m_phi_t=cap["mism"].phi_t, m_e_t=cap["mism"].e_t,
               corr=cap["corr"], dcorr=cap["dcorr"], fields=cap["fields"],
               far=cap["far"], over=part.over, far_idx=part.far,
               img_pos=part.image_positions, img_str=part.image_strengths,
               img_src=part.image_source, img_wall=part.image_wall,
               pair_e=eidx.astype(np.int32), pair_s=sidx.astype(np.int32))
    return out


def params_record(p):
    d = p.as_dict()
    return {k: (repr(v) if isinstance(v, float) else v) for k, v in d.items()}


def main():
    warnings.simplefilter("ignore")
    meta = {"reference": "slabewald %s" % sw.__version__,
            "numpy": np.__version__}
    import scipy
    meta["scipy"] = scipy.__version__

    # ---- planner goldens -------------------------------------------------
    plans = {}
    for name in ("c1", "c2", "c3", "c4", "c5"):
        plans[name] = params_record(ref_problem(name, N=4)[1])
    pub = sw.SlabGeometry(2.0, 2.0, 0.75, 1.0, 1 / 20, 1 / 50)
    for xi in (4.3, 9.2, 12.2, 26.0):
        p = sw.plan_grid(pub, 0.025, 5e-4, xi=xi, h_min=4.5 * 0.025,
                         strict=False)
        plans["published_xi_%g" % xi] = params_record(p)
    for L in (28.0, 32.0):
        geo = sw.SlabGeometry(L, L, 2.0, 1.0, 0.5, 0.2)
        p = sw.plan_grid(geo, 0.01, 1e-4, xi=3.0177, h_min=0.01,
                         strict=False)
        plans["freespace_L%g" % L] = params_record(p)
    cut = {}
    for xi, g_w, delta in ((1.0, 0.0, 1e-4), (3.0, 0.01, 1e-4),
                           (1.0, 0.5 / np.sqrt(3.0), 1e-4), (6.8, 0.01, 1e-4),
                           (47.21, 0.0027, 1e-4), (2.0, 0.05, 5e-4)):
        cut["%r_%r_%r" % (xi, g_w, delta)] = repr(sw.tune_cutoff(xi, g_w,
                                                                 delta))
    with open(os.path.join(HERE, "params.json"), "w") as fh:
        json.dump({"meta": meta, "plans": plans, "tune_cutoff": cut}, fh,
                  indent=1, sort_keys=True)
    print("params.json")

    # ---- Chebyshev / BVP primitives --------------------------------------
    prim = {}
    for n in (32, 107, 158, 258):
        prim["nodes_%d" % n] = sw_cheb.cheb_nodes(n, -0.3, 1.7)
        prim["ccw_%d" % n] = sw_cheb.clenshaw_curtis_weights(n, -0.3, 1.7)
    rng = np.random.default_rng(5)
    for n in (33, 107):
        f = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        prim["f_%d" % n] = f
        plan = sw_bvp.BvpPlan(n, -0.4, 1.6)
        ks = np.array([0.7, 3.0, 25.0, 300.0])
        fac = sw_bvp.BvpFactor(plan, ks)
        batch = np.tile(f, (ks.size, 1))
        prim["k_%d" % n] = ks
        prim["y_ref1_%d" % n] = fac.solve(batch, refine=1)
        prim["y_ref0_%d" % n] = fac.solve(batch, refine=0)
        prim["y_k0_%d" % n] = sw_bvp.solve_k0_dirichlet(plan, f)
        prim["dct_%d" % n] = sw_cheb.cheb_transform(f.real)
        prim["idct_%d" % n] = sw_cheb.cheb_inverse(f.real)
        prim["deriv_%d" % n] = sw_cheb.cheb_derivative(f, -0.4, 1.6)
    np.savez_compressed(os.path.join(HERE, "primitives.npz"), **prim)
    print("primitives.npz")

    # ---- end-to-end solves -----------------------------------------------
    cases = {}
    print("c1")
    s, p = ref_problem("c1")
    cases["c1"] = outputs(run_solve(s, p))
    print("c2")
    s, p = ref_problem("c2")
    cases["c2"] = outputs(run_solve(s, p))
    print("c3")
    s, p = ref_problem("c3")
    cases["c3"] = outputs(run_solve(s, p))
    # variants on the C2 box with 256 charges
    print("variants")
    s, p = ref_problem("c2", N=256)
    cases["c2n256"] = outputs(run_solve(s, p))
    cases["c2n256_refine0"] = outputs(run_solve(s, p, refine=0))
    cases["c2n256_noforce"] = outputs(run_solve(s, p, need_forces=False))
    cases["c2n256_nopot"] = outputs(run_solve(s, p, need_potential=False))
    cases["c2n256_selfsub"] = outputs(run_solve(s, p, subtract_self=True))
    cases["c2n256_nocorr"] = outputs(run_solve(s, p,
                                               include_correction=False))
    s, p = ref_problem("c2", N=256, eps_b=1.0, eps_t=1.0)
    cases["c2n256_nojump"] = outputs(run_solve(s, p))
    cases["c2n256_general"] = outputs(run_solve(s, p, force_general=True))
    s, p = ref_problem("c2", N=256, eps_b=1.0, eps_t=1.0,
                       surface=sw.SurfaceCharge.uniform(0.3, -0.3))
    cases["c2n256_nojump_sigma"] = outputs(run_solve(s, p))
    s, p = ref_problem("c3", N=256,
                       surface=sw.SurfaceCharge.gaussian(0.3, 1.5, -1.5))
    cases["c3n256_gauss_sigma"] = outputs(run_solve(s, p))
    s, p = ref_problem("c3", N=512, eps_b=0.0, eps_t=40.0)
    cases["c3n512_vacuum_metal"] = outputs(run_solve(s, p))
    # moved positions through the positions= override (BD style)
    s, p = ref_problem("c2", N=256)
    moved = s.positions + 0.01 * np.random.default_rng(3).standard_normal(
        s.positions.shape)
    moved[:, 2] = np.clip(moved[:, 2], 0.1, 0.9)
    out = outputs(run_solve(s, p, positions=moved))
    out["positions"] = moved
    cases["c2n256_moved"] = out
    # no-split reference (xi = inf) on a small problem
    geo = sw.SlabGeometry(1.0, 1.0, 0.5, 1.0, 0.2, 3.0)
    pos = np.array([[0.3, 0.4, 0.2], [0.7, 0.45, 0.3], [0.5, 0.8, 0.25],
                    [0.1, 0.1, 0.35]])
    q = np.array([1.0, -1.0, 1.0, -1.0])
    s = sw.ChargeSystem(geo, pos, q, 0.05)
    p = sw_ref.unsplit_params(geo, 0.05)
    t0 = time.time()
    res = sw.SlabSolver(s, p).solve(subtract_self=True)
    print("   unsplit %.2fs grid %dx%dx%d" % (time.time() - t0, p.Nx, p.Ny,
                                             p.Nz))
    out = outputs(res)
    out["positions"], out["charges"] = pos, q
    cases["unsplit4"] = out
    np.savez_compressed(os.path.join(HERE, "solves.npz"),
                        **{"%s__%s" % (c, k): v for c, d in cases.items()
                           for k, v in d.items()})
    print("solves.npz")

    # ---- per-stage intermediates on a tiny jump case ---------------------
    geo = sw.SlabGeometry(1.5, 1.5, 1.0, 1.0, 0.05, 0.02)
    rng = np.random.default_rng(11)
    n = 48
    pos = np.column_stack([rng.uniform(0, 1.5, n), rng.uniform(0, 1.5, n),
                           rng.uniform(0.13, 0.87, n)])
    pos[:6, 2] = [0.14, 0.2, 0.25, 0.8, 0.75, 0.86]     # wall-overlapping
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    s = sw.ChargeSystem(geo, pos, q, 0.03)
    p = sw.plan_grid(geo, 0.03, 1e-4, Nxy=24)
    print("tiny grid %dx%dx%d" % (p.Nx, p.Ny, p.Nz))
    st = capture_stages(s, p)
    st["positions"], st["charges"] = pos, q
    st["plan"] = np.array([p.Nx, p.Nz])
    np.savez_compressed(os.path.join(HERE, "stages_tiny.npz"), **st)
    # pair list + partition for C3 (membership is checked bit-exactly)
    s, p = ref_problem("c3")
    part = sw.build_partition(s.positions, s.charges, s.geometry, p)
    np.savez_compressed(os.path.join(HERE, "partition_c3.npz"),
                        over=part.over.astype(np.int32),
                        img_src=part.image_source.astype(np.int32),
                        img_wall=part.image_wall.astype(np.int8))
    s, p = ref_problem("c2", N=512)
    nf = sw_slab.NearField(s.positions, s.charges, s.geometry, p)
    eidx, sidx, d, r = nf._pairs(s.positions, p.r_cut)
    np.savez_compressed(os.path.join(HERE, "pairs_c2n512.npz"),
                        e=eidx.astype(np.int32), s=sidx.astype(np.int32))
    print("done")


if __name__ == "__main__":
    main()
