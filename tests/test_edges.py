"""Edge cases against reference-generated goldens (tests/golden/edges.npz,
made by tests/golden/make_edges.py): coincident charges, charges on grid
nodes, a pair at exactly the cutoff, charges on the walls (coincident with
their images), charges on the periodic edge, a single (non-neutral) charge
and an empty system.  The oracle is checked on CPU, the CUDA path on GPU."""

import os

import numpy as np
import pytest

from oracle import slab_oracle as O
import _edge_cases as EC
from paper_2101_07088_b200.geometry import ChargeSystem, SlabGeometry
from paper_2101_07088_b200.params import plan_grid
from _golden import rel_l2

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "edges.npz"))
OK = [c for c in EC.CASES if c + "__phi" in GOLD.files]
RAISES = {c: str(GOLD[c + "__error"]) for c in EC.CASES if c + "__error" in GOLD.files}


def _problem(name):
    geo_args, pos, q, g_w, delta, nxy = EC.build(name)
    geo = SlabGeometry(*geo_args)
    return ChargeSystem(geo, pos, q, g_w), plan_grid(geo, g_w, delta, Nxy=nxy)


def _check(phi, E, U, B_i, name, tol):
    assert rel_l2(phi, GOLD[name + "__phi"]) < tol, name
    assert rel_l2(E, GOLD[name + "__E"]) < tol, name
    g_u = float(GOLD[name + "__U"])
    assert abs(U - g_u) <= tol * max(1.0, abs(g_u)), name
    g_b = float(GOLD[name + "__B_i"])
    assert abs(B_i - g_b) <= tol * max(1.0, abs(g_b)), name


def test_edge_goldens_present():
    assert set(OK) == {"coincident", "on_nodes", "at_cutoff", "walls",
                       "periodic_edge", "empty"}
    assert RAISES == {"single": "FloatingPointError"}


@pytest.mark.parametrize("name", OK)
def test_oracle_edges(name):
    system, params = _problem(name)
    phi, E, U, diag = O.OracleSlabSolver(system, params).solve()
    _check(phi, E, U, diag["B_i"], name, 1e-12)
    nf = O.NearSources(system.positions, system.charges, system.geometry,
                       params)
    if system.charges.size:
        e = nf.pairs(system.positions, params.r_cut)[0]
        assert len(e) == int(GOLD[name + "__npairs"])


def test_oracle_single_charge_raises():
    system, params = _problem("single")
    with pytest.raises(FloatingPointError):
        O.OracleSlabSolver(system, params).solve()


@pytest.mark.gpu
@pytest.mark.parametrize("name", OK)
def test_gpu_edges(name):
    from paper_2101_07088_b200.slab import SlabSolver
    system, params = _problem(name)
    res = SlabSolver(system, params).solve()
    _check(res.phi_bar, res.E_bar, res.U, res.diagnostics["B_i"], name, 1e-10)
    assert res.diagnostics["n_pairs"] == int(GOLD[name + "__npairs"])


@pytest.mark.gpu
def test_gpu_single_charge_raises():
    from paper_2101_07088_b200.slab import SlabSolver
    system, params = _problem("single")
    with pytest.raises(FloatingPointError):
        SlabSolver(system, params).solve()


