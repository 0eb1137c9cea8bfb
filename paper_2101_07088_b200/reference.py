"""Solver-level accuracy harness of the reference (``slabewald.reference``,
reference.py:78-147) over the GPU solver: the no-splitting (xi -> infinity)
solve, the energy-force work check and the L -> infinity extrapolation, as
used by the reference's validate suites.  The 400-image open-slab oracle
(``free_space_slab_reference``) is a host numpy computation of the reference
and is not reproduced here."""

import math
from dataclasses import dataclass

import numpy as np

from .params import EwaldParams


def richardson_infinite_box(val_small, l_small, val_big, l_big):
    """Extrapolate to L = infinity assuming an O(1/L) finite-size term
    (reference.py:78-80)."""
    return (l_big * val_big - l_small * val_small) / (l_big - l_small)


def unsplit_params(geometry, g_w, resolve=2.0, n_sigma=6.0, max_points=2**27):
    """Grid parameters for the no-splitting reference (reference.py:83-105):
    spacing g_w / resolve, bare charge Gaussian truncated at n_sigma, no
    near field."""
    h = g_w / resolve
    nx = max(int(round(geometry.Lx / h)), 4)
    ny = max(int(round(geometry.Ly / h)), 4)
    h_xy = geometry.Lx / nx
    h_e = n_sigma * g_w
    z0, z1 = -3.0 * h_e, geometry.H + 3.0 * h_e
    nz = int(math.ceil(math.pi * (z1 - z0) / (2.0 * h_xy)))
    if nx * ny * nz > max_points:
        raise MemoryError("reference grid %dx%dx%d exceeds the guard" % (nx, ny, nz))
    return EwaldParams(
        xi=np.inf, g_w=g_w, g_t=g_w, delta=0.0,
        n_g=int(math.ceil(2.0 * h_e / h_xy)), n_sigma=n_sigma, h_xy=h_xy,
        H_E=h_e, r_nf=0.0, r_cut=0.0, k_max=math.pi / h_xy,
        Nx=nx, Ny=ny, Nz=nz, z0=z0, z1=z1, h_min=n_sigma * g_w)


def no_split_reference(system, resolve=2.0, n_sigma=6.0, max_points=2**27, threads=1,
                       **solve_kw):
    """Solve without Ewald splitting on a g_w-resolving grid
    (reference.py:108-113)."""
    from .slab import SlabSolver
    params = unsplit_params(system.geometry, system.g_w, resolve, n_sigma, max_points)
    solver = SlabSolver(system, params, threads=threads)
    try:
        return solver.solve(**solve_kw)
    finally:
        solver.close()


@dataclass
class WorkCheck:
    W1: float
    W2: float
    reldiff: float
    degenerate: bool = False


def work_check(solver, delta0=1e-4, direction=None, rng=None, subtract_self=False):
    """Energy-force consistency along per-charge unit displacements
    (reference.py:124-147): W1 the centred difference of U, W2 = sum F.dX."""
    pos = solver.system.positions
    n = pos.shape[0]
    if direction is None:
        rng = np.random.default_rng(rng)
        direction = rng.standard_normal((n, 3))
        direction /= np.linalg.norm(direction, axis=1, keepdims=True)
    res = solver.solve(positions=pos, subtract_self=subtract_self)
    w2 = float(np.sum(res.forces * direction))
    up = solver.solve(positions=pos + 0.5 * delta0 * direction, need_forces=False,
                      subtract_self=subtract_self).U
    dn = solver.solve(positions=pos - 0.5 * delta0 * direction, need_forces=False,
                      subtract_self=subtract_self).U
    w1 = -(up - dn) / delta0
    if abs(w1) < 1e-14:
        return WorkCheck(w1, w2, 0.0, degenerate=True)
    return WorkCheck(w1, w2, abs(w1 - w2) / abs(w1))


__all__ = ["richardson_infinite_box", "unsplit_params", "no_split_reference",
           "WorkCheck", "work_check"]
