"""Planner parity: plan_grid / tune_cutoff reproduce the reference's values
bit for bit (golden params.json made by the reference), plus the
reference's own published-size tests (reference tests/test_params.py)."""

import warnings

import numpy as np
import pytest

from paper_2101_07088_b200 import workloads as W
from paper_2101_07088_b200.geometry import SlabGeometry
from paper_2101_07088_b200.params import (ACCURACY_PROFILES, ConstraintError,
                                          plan_grid, tune_cutoff)
from _golden import plans

FIELDS = ("xi", "g_w", "g_t", "delta", "n_g", "n_sigma", "h_xy", "H_E", "r_nf",
          "r_cut", "k_max", "Nx", "Ny", "Nz", "z0", "z1", "h_min", "n_img")


def _same(rec, p):
    for f in FIELDS:
        want = rec[f]
        got = getattr(p, f)
        if isinstance(want, str):
            assert repr(float(got)) == want, (f, got, want)
        else:
            assert got == want, (f, got, want)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_workload_plans_bit_identical(name):
    _same(plans()["plans"][name], W.build(name, N=4)[1])


def test_published_plans_bit_identical():
    pub = SlabGeometry(2.0, 2.0, 0.75, 1.0, 1 / 20, 1 / 50)
    for xi in (4.3, 9.2, 12.2, 26.0):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            p = plan_grid(pub, 0.025, 5e-4, xi=xi, h_min=4.5 * 0.025,
                          strict=False)
        _same(plans()["plans"]["published_xi_%g" % xi], p)
    for L in (28.0, 32.0):
        geo = SlabGeometry(L, L, 2.0, 1.0, 0.5, 0.2)
        p = plan_grid(geo, 0.01, 1e-4, xi=3.0177, h_min=0.01, strict=False)
        _same(plans()["plans"]["freespace_L%g" % L], p)


def test_tune_cutoff_bit_identical():
    for key, want in plans()["tune_cutoff"].items():
        xi, g_w, delta = (float(v.replace("np.float64(", "").rstrip(")"))
                          for v in key.split("_"))
        assert repr(tune_cutoff(xi, g_w, delta)) == want


def test_profiles_and_published_sizes():
    assert ACCURACY_PROFILES[1e-4] == (12, 1.4)
    assert ACCURACY_PROFILES[5e-4] == (10, 1.2)
    geo = SlabGeometry(2.0, 2.0, 0.75, 1.0, 1 / 20, 1 / 50)
    expect = {4.3: (20, 59, 0.5), 9.2: (40, 71, 0.25), 12.2: (50, 77, 0.20),
              26.0: (76, 92, 0.13)}
    for xi, (nxy, nz, h_e) in expect.items():
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            p = plan_grid(geo, 0.025, 5e-4, xi=xi, h_min=4.5 * 0.025,
                          strict=False)
        assert (p.Nx, p.Ny, p.Nz) == (nxy, nxy, nz)
        assert abs(p.H_E - h_e) < 0.01


def test_constraints_and_argument_errors():
    geo = SlabGeometry(2.0, 2.0, 0.75, 1.0, 1 / 20, 1 / 50)
    with pytest.raises(ConstraintError, match="efficiency"):
        plan_grid(geo, 0.025, 5e-4, xi=15.0, h_min=0.1)
    with pytest.warns(UserWarning, match="efficiency"):
        p = plan_grid(geo, 0.025, 5e-4, xi=15.0, h_min=0.1, strict=False)
    assert not all(ok for _, ok, _ in p.constraints)
    with pytest.raises(ConstraintError, match="far_field_images"):
        plan_grid(geo, 0.025, 5e-4, xi=4.3, h_min=4.5 * 0.025)
    with pytest.raises(ValueError):
        plan_grid(SlabGeometry(2.0, 2.0, 1.0, 1.0), 0.01, 1e-4)
    with pytest.raises(ValueError):
        plan_grid(SlabGeometry(2.0, 2.0, 1.0, 1.0), 0.01, 1e-5, Nxy=32)
    p = plan_grid(SlabGeometry(4.0, 4.0, 2.0, 1.0), 0.02, 1e-4, xi=4.0,
                  h_min=0.2)
    assert abs(p.g_t - np.hypot(1 / 8.0, 0.02)) < 1e-15
    assert p.as_dict()["constraints"][0]["name"] == "efficiency"
