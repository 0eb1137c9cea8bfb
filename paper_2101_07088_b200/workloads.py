"""Synthetic workloads C1-C5 of the benchmark plan.

Each workload is a plain description (box, permittivities, g_w, planner
inputs, charge count and seed) so the same inputs can be rebuilt by the
GPU product, by the CPU oracle and, in the build container, by the
reference package itself (``tests/golden/make_golden.py``).

Inputs: ``np.random.default_rng(seed)``; x, y ~ U[0, L); z ~ U[n_sigma g_w,
H - n_sigma g_w]; charges alternate +1/-1 by index (electroneutral for even
N); eps = 1 inside.
"""

import math

import numpy as np

from .geometry import ChargeSystem, SlabGeometry, SurfaceCharge
from .params import ACCURACY_PROFILES, EwaldParams, plan_grid, tune_cutoff
from .kernels import split_widths

# name -> description.  "Nxy" feeds plan_grid; "hand" builds EwaldParams
# directly (C1's 32^3 grid is below what the planner emits for delta=1e-4).
WORKLOADS = {
    "c1": dict(L=8.0, H=4.0, eps_b=1.0, eps_t=1.0, g_w=0.1, delta=1e-4,
               hand=dict(h=0.25, g_t=0.35, Nz=32), N=2, seed=None),
    "c2": dict(L=2.0, H=1.0, eps_b=0.05, eps_t=1.0, g_w=0.02, delta=1e-4,
               Nxy=64, N=2048, seed=0),
    "c3": dict(L=2.0, H=1.0, eps_b=0.05, eps_t=0.02, g_w=0.005, delta=1e-4,
               Nxy=128, N=32768, seed=0),
    "c4": dict(L=2.0, H=1.0, eps_b=0.05, eps_t=0.05,
               g_w=0.25 * 1.4 * 2.0 / 256, delta=1e-4, Nxy=256, N=1 << 20,
               seed=0),
    # C4 density and grid spacing in a 0.5 x 0.5 box: the same h, Nz = 258,
    # ~575 near pairs per charge, at a size the CPU reference finishes
    "c4d": dict(L=0.5, H=1.0, eps_b=0.05, eps_t=0.05,
                g_w=0.25 * 1.4 * 2.0 / 256, delta=1e-4, Nxy=64, N=1 << 16,
                seed=0),
    "c5": dict(L=8.0, H=1.0, eps_b=0.05, eps_t=0.05,
               g_w=0.25 * 1.4 * 2.0 / 256, delta=1e-4, Nxy=1024,
               N=1 << 24, seed=0),
    # the paper's performance study:
    # 2e4 charges, H = 50, L = 185, g_w = a/4 (a = 1), optimum N_xy = 88
    "paper": dict(L=185.0, H=50.0, eps_b=0.05, eps_t=0.05, g_w=0.25,
                  delta=1e-4, Nxy=88, N=20000, seed=0),
}


def hand_params(desc):
    """EwaldParams for a hand-specified grid (C1), derived like the planner
    but with the given spacing, g_t and Nz."""
    hd = desc["hand"]
    g_w, delta = desc["g_w"], desc["delta"]
    n_g, factor = ACCURACY_PROFILES[delta]
    h, g_t = hd["h"], hd["g_t"]
    xi = 0.5 / math.sqrt(g_t**2 - g_w**2)
    H_E = 0.5 * n_g * h
    n_sigma = n_g / (2.0 * factor)
    r_nf = tune_cutoff(xi, g_w, delta)
    nxy = int(round(desc["L"] / h))
    return EwaldParams(xi=xi, g_w=g_w, g_t=g_t, delta=delta, n_g=n_g,
                       n_sigma=n_sigma, h_xy=h, H_E=H_E, r_nf=r_nf,
                       r_cut=r_nf + n_sigma * g_w, k_max=math.pi / h,
                       Nx=nxy, Ny=nxy, Nz=hd["Nz"], z0=-3.0 * H_E,
                       z1=desc["H"] + 3.0 * H_E, h_min=n_sigma * g_w)


def make_inputs(desc, N=None):
    """(positions, charges) of a workload; ``N`` overrides the count."""
    n = desc["N"] if N is None else int(N)
    L, H = desc["L"], desc["H"]
    if desc["seed"] is None:                      # C1: the fixed pair
        pos = np.array([[L / 2 - 0.5, L / 2, H / 2],
                        [L / 2 + 0.5, L / 2, H / 2]])[:n]
        return pos, np.array([1.0, -1.0])[:n]
    n_g, factor = ACCURACY_PROFILES[desc["delta"]]
    margin = n_g / (2.0 * factor) * desc["g_w"]
    rng = np.random.default_rng(desc["seed"])
    pos = np.empty((n, 3))
    pos[:, 0] = rng.uniform(0.0, L, n)
    pos[:, 1] = rng.uniform(0.0, L, n)
    pos[:, 2] = rng.uniform(margin, H - margin, n)
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    return pos, q


def build(name, N=None, surface=None, **override):
    """(system, params) of workload ``name`` for the product API."""
    desc = dict(WORKLOADS[name])
    desc.update(override)
    geo = SlabGeometry(desc["L"], desc["L"], desc["H"], 1.0, desc["eps_b"],
                       desc["eps_t"])
    pos, q = make_inputs(desc, N)
    system = ChargeSystem(geo, pos, q, desc["g_w"], surface)
    if "hand" in desc:
        params = hand_params(desc)
    else:
        params = plan_grid(geo, desc["g_w"], desc["delta"], Nxy=desc["Nxy"])
    return system, params


__all__ = ["WORKLOADS", "build", "make_inputs", "hand_params",
           "SurfaceCharge", "split_widths"]
