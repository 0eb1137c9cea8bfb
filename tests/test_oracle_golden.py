"""Pin the CPU oracle against fixtures produced by the reference itself.

The oracle (``oracle/slab_oracle.py``) is what the GPU parity tests check
against on the GPU box, so it must first agree with the reference here.
Tolerances: stencil/partition/pair membership exact; grids, coefficients
and per-charge outputs within 1e-12 relative L2 (same libraries, rounding
differences only).
"""

import numpy as np
import pytest

from oracle import slab_oracle as O
from paper_2101_07088_b200 import workloads as W
from paper_2101_07088_b200.geometry import (ChargeSystem, SlabGeometry,
                                            SurfaceCharge)
from paper_2101_07088_b200.params import plan_grid
from _golden import primitives, rel_l2, solves, stages

TOL = 1e-12


@pytest.fixture(scope="module")
def gold():
    return solves()


def _check(out, g, tol=TOL, forces=True):
    phi, E, U, diag = out
    assert rel_l2(phi, g["phi"]) < tol
    if forces:
        assert rel_l2(E, g["E"]) < tol
    assert abs(U - g["U"]) <= tol * max(1.0, abs(g["U"]))
    assert abs(diag["B_i"] - g["B_i"]) <= tol * max(1.0, abs(g["B_i"]))
    assert abs(diag["k0"]["A_i"] - g["A_i"]) <= 1e-10 * max(1.0,
                                                            abs(g["A_i"]))


def test_primitives_match_reference():
    g = primitives()
    for n in (32, 107, 158, 258):
        assert np.array_equal(O.cheb_nodes(n, -0.3, 1.7), g["nodes_%d" % n])
        assert np.array_equal(O.cc_weights(n, -0.3, 1.7), g["ccw_%d" % n])
    for n in (33, 107):
        f = g["f_%d" % n]
        bank = O.BvpBank(n, -0.4, 1.6, g["k_%d" % n])
        rows = np.arange(4)
        batch = np.tile(f, (4, 1))
        assert rel_l2(bank.solve(batch, rows, 1), g["y_ref1_%d" % n]) < 1e-14
        assert rel_l2(bank.solve(batch, rows, 0), g["y_ref0_%d" % n]) < 1e-14
        assert rel_l2(bank.solve_k0(f), g["y_k0_%d" % n]) < 1e-14
        assert rel_l2(O.cheb_coeffs(f.real), g["dct_%d" % n]) < 1e-15
        assert rel_l2(O.cheb_values(f.real), g["idct_%d" % n]) < 1e-15
        assert rel_l2(O.cheb_deriv(f, -0.4, 1.6), g["deriv_%d" % n]) < 1e-15


def test_stages_tiny_case():
    g = stages()
    geo = SlabGeometry(1.5, 1.5, 1.0, 1.0, 0.05, 0.02)
    sysm = ChargeSystem(geo, g["positions"], g["charges"], 0.03)
    par = plan_grid(geo, 0.03, 1e-4, Nxy=24)
    cap = {}
    out = O.OracleSlabSolver(sysm, par).solve(capture=cap)
    part = cap["partition"]
    assert np.array_equal(part["over"], g["over"])
    assert np.array_equal(part["far"], g["far_idx"])
    assert np.array_equal(part["image_source"], g["img_src"])
    assert np.array_equal(part["image_wall"], g["img_wall"])
    assert np.array_equal(part["image_positions"], g["img_pos"])
    assert rel_l2(cap["rho_over"], g["rho_over"]) < TOL
    assert rel_l2(cap["rho_in"], g["rho_over"] + g["rho_far"]) < TOL
    assert rel_l2(cap["psi_o"], g["psi_o"]) < TOL
    assert rel_l2(cap["psi_i"], g["psi_i"]) < TOL
    for key in ("phi_b", "e_b", "phi_t", "e_t"):
        assert rel_l2(cap["mismatch"][key], g["m_" + key]) < TOL
    assert rel_l2(cap["corr"], g["corr"]) < TOL
    assert rel_l2(cap["dcorr"], g["dcorr"]) < TOL
    assert rel_l2(cap["fields"], g["fields"]) < TOL
    nf = O.NearSources(sysm.positions, sysm.charges, geo, par)
    ti, sj, _, _ = nf.pairs(sysm.positions, par.r_cut)
    assert np.array_equal(ti, g["pair_e"]) and np.array_equal(sj, g["pair_s"])
    _check(out, g)


@pytest.mark.parametrize("case", ["c1", "c2"])
def test_workload_solves(gold, case):
    system, params = W.build(case)
    _check(O.oracle_solve(system, params), gold[case])


@pytest.mark.slow
def test_workload_c3(gold):
    system, params = W.build("c3")
    _check(O.oracle_solve(system, params), gold["c3"])


VARIANTS = {
    "c2n256": ("c2", {}, {}, None),
    "c2n256_refine0": ("c2", {}, {"refine": 0}, None),
    "c2n256_noforce": ("c2", {}, {"need_forces": False}, None),
    "c2n256_nopot": ("c2", {}, {"need_potential": False}, None),
    "c2n256_selfsub": ("c2", {}, {"subtract_self": True}, None),
    "c2n256_nocorr": ("c2", {}, {"include_correction": False}, None),
    "c2n256_nojump": ("c2", {"eps_b": 1.0, "eps_t": 1.0}, {}, None),
    "c2n256_general": ("c2", {"eps_b": 1.0, "eps_t": 1.0},
                       {"force_general": True}, None),
    "c2n256_nojump_sigma": ("c2", {"eps_b": 1.0, "eps_t": 1.0}, {},
                            ("uniform", (0.3, -0.3))),
    "c3n256_gauss_sigma": ("c3", {}, {}, ("gaussian", (0.3, 1.5, -1.5))),
    "c3n512_vacuum_metal": ("c3", {"eps_b": 0.0, "eps_t": 40.0}, {}, None),
}


def variant_problem(case):
    base, over, kw, surf = VARIANTS[case]
    n = 512 if case.startswith("c3n512") else 256
    surface = None
    if surf is not None:
        surface = getattr(SurfaceCharge, surf[0])(*surf[1])
    system, params = W.build(base, N=n, surface=surface, **over)
    return system, params, dict(kw)


@pytest.mark.parametrize("case", sorted(VARIANTS))
def test_variants(gold, case):
    system, params, kw = variant_problem(case)
    refine = kw.pop("refine", 1)
    out = O.OracleSlabSolver(system, params, refine=refine).solve(**kw)
    _check(out, gold[case], forces=kw.get("need_forces", True))


def test_positions_override(gold):
    g = gold["c2n256_moved"]
    system, params = W.build("c2", N=256)
    out = O.OracleSlabSolver(system, params).solve(positions=g["positions"])
    _check(out, g)


def test_unsplit_no_near_field(gold):
    g = gold["unsplit4"]
    geo = SlabGeometry(1.0, 1.0, 0.5, 1.0, 0.2, 3.0)
    system = ChargeSystem(geo, g["positions"], g["charges"], 0.05)
    from paper_2101_07088_b200.params import EwaldParams
    import math
    g_w, h_e = 0.05, 6.0 * 0.05
    h = g_w / 2.0
    nx = int(round(1.0 / h))
    params = EwaldParams(xi=np.inf, g_w=g_w, g_t=g_w, delta=0.0,
                         n_g=int(math.ceil(2.0 * h_e / (1.0 / nx))),
                         n_sigma=6.0, h_xy=1.0 / nx, H_E=h_e, r_nf=0.0,
                         r_cut=0.0, k_max=math.pi / (1.0 / nx), Nx=nx, Ny=nx,
                         Nz=int(math.ceil(math.pi * (0.5 + 6 * h_e)
                                          / (2.0 * (1.0 / nx)))),
                         z0=-3.0 * h_e, z1=0.5 + 3.0 * h_e, h_min=6.0 * g_w)
    out = O.OracleSlabSolver(system, params).solve(subtract_self=True)
    _check(out, g)
