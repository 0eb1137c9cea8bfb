"""The reference's solver-level accuracy suites on the GPU, against the
reference's own results (tests/golden/make_checks.py): xi-independence vs
the no-splitting solve (validate.py:140-170, PAPER Table 3) and the
energy-force work check with charged Gaussian walls (validate.py:175-203,
PAPER Table 5)."""

import os
import warnings

import numpy as np
import pytest

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "checks.npz"))


def test_unsplit_params_match_reference_formula():
    from paper_2101_07088_b200 import SlabGeometry
    from paper_2101_07088_b200.reference import unsplit_params
    p = unsplit_params(SlabGeometry(2.0, 2.0, 0.75, 1.0, 1 / 20, 1 / 50), 0.025)
    assert (p.Nx, p.Ny) == (160, 160) and p.xi == np.inf and p.r_cut == 0.0


@pytest.mark.gpu
def test_xi_independence_matches_reference():
    from paper_2101_07088_b200 import ChargeSystem, SlabGeometry, plan_grid
    from paper_2101_07088_b200.reference import no_split_reference
    from paper_2101_07088_b200.slab import SlabSolver
    H, L, g_w, n_charges = 0.75, 2.0, 0.025, 100
    geo = SlabGeometry(L, L, H, eps=1.0, eps_b=1 / 20, eps_t=1 / 50)
    rng = np.random.default_rng(7)
    xis = tuple(G["xi_values"])
    errors = {xi: [] for xi in xis}
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        params = {xi: plan_grid(geo, g_w, 5e-4, xi=xi, h_min=4.5 * g_w, strict=False)
                  for xi in xis}
        for _ in range(3):
            pos = np.column_stack([rng.uniform(0, L, n_charges), rng.uniform(0, L, n_charges),
                                   rng.uniform(4.5 * g_w, H - 4.5 * g_w, n_charges)])
            q = np.where(np.arange(n_charges) % 2 == 0, 1.0, -1.0)
            system = ChargeSystem(geo, pos, q, g_w)
            ref = no_split_reference(system, resolve=2.0, n_sigma=6.0)
            scale = np.mean(np.linalg.norm(ref.E_bar, axis=1))
            for xi in xis:
                res = SlabSolver(system, params[xi]).solve()
                errors[xi].append((res.E_bar - ref.E_bar) / scale)
    std = np.array([np.concatenate([e.ravel() for e in errors[xi]]).std() for xi in xis])
    assert np.all(std <= 1e-4)
    assert np.allclose(std, G["xi_std"], rtol=1e-6, atol=0)


@pytest.mark.gpu
def test_work_check_matches_reference():
    from paper_2101_07088_b200 import ChargeSystem, SlabGeometry, SurfaceCharge, plan_grid
    from paper_2101_07088_b200.reference import work_check
    from paper_2101_07088_b200.slab import SlabSolver
    H, L, n = 1.0, 2.0, 10
    geo = SlabGeometry(L, L, H, eps=1.0, eps_b=1 / 20, eps_t=1 / 50)
    rng = np.random.default_rng(11)
    pos = np.column_stack([rng.uniform(0, L, n), rng.uniform(0, L, n),
                           rng.uniform(0.045, H - 0.045, n)])
    q = np.tile([1.0, -1.0], n // 2)
    surf = SurfaceCharge.gaussian(s=0.2, charge_b=0.5, charge_t=-0.5)
    direction = np.random.default_rng(0).standard_normal((n, 3))
    direction /= np.linalg.norm(direction, axis=1, keepdims=True)
    rel, w1, w2 = [], [], []
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for g_w in (1e-2, 1e-3, 1e-4, 1e-10):
            system = ChargeSystem(geo, pos, q, g_w, surf)
            params = plan_grid(geo, g_w, 1e-4, xi=6.8, h_min=0.045, strict=False)
            wc = work_check(SlabSolver(system, params), delta0=1e-4, direction=direction,
                            subtract_self=True)
            assert not wc.degenerate
            rel.append(wc.reldiff); w1.append(wc.W1); w2.append(wc.W2)
    assert np.all(np.array(rel) <= 1e-3)
    assert np.allclose(w2, G["wc_W2"], rtol=1e-9, atol=0)
    # W1 is a centred difference of U over 1e-4 moves: U to 1e-13 relative
    # gives W1 to ~1e-8 relative
    assert np.allclose(w1, G["wc_W1"], rtol=1e-6, atol=0)
