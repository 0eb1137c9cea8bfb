"""TEST INFRASTRUCTURE — numpy restatement of the reference's triply periodic
twin, the checker for se_tp_* on machines without the
reference.  Only tests, ``smoke()`` and bench's CPU legs may call it.

Follows solve_triply_periodic (dpsolver.py:221-249), PeriodicGrid3d
(gridops.py:136-192) and TriplyPeriodicSolver (bd.py:297-355); pinned against
tests/golden/tp.npz (made by the reference itself, tests/golden/make_tp.py).
Pair search is brute force over all pairs (small N only), full minimum image.
"""

import math

import numpy as np

from .slab_oracle import (FOUR_PI, _axis_uniform, _gauss, d_erf_over_r,
                          kernel_widths, wavenumbers)

ACCURACY = {1e-4: (12, 1.4), 5e-4: (10, 1.2)}        # params.py ACCURACY_PROFILES


def poisson(rho, eps, L, with_field=False):
    """dpsolver.py:221-249 with numpy.fft."""
    n = rho.shape
    rho_hat = np.fft.fftn(rho)
    kx, ky = wavenumbers(n[0], n[1], L[0], L[1])
    kz = 2.0 * np.pi * np.fft.fftfreq(n[2], d=1.0 / n[2]) / L[2]
    k2 = kx[:, None, None] ** 2 + ky[None, :, None] ** 2 + kz[None, None, :] ** 2
    k2[0, 0, 0] = 1.0
    phi_hat = rho_hat / (eps * k2)
    phi_hat[0, 0, 0] = 0.0
    phi = np.fft.ifftn(phi_hat).real
    if not with_field:
        return phi
    e = np.empty((3,) + n)
    for ax, kv in enumerate((kx, ky, kz)):
        kv = kv.copy()
        if n[ax] % 2 == 0:
            kv[n[ax] // 2] = 0.0
        shp = [1, 1, 1]
        shp[ax] = n[ax]
        e[ax] = np.fft.ifftn(-1j * kv.reshape(shp) * phi_hat).real
    return phi, e


def _stencils(pos, h, n, width, radius):
    out = []
    for ax in range(3):
        idx, off, keep = _axis_uniform(pos[:, ax], h[ax], n[ax], radius)
        out.append((idx, _gauss(off, keep, width)))
    return out


def spread(pos, q, L, n, width, radius):
    """gridops.py:155-174 (one charge at a time)."""
    h = [L[a] / n[a] for a in range(3)]
    out = np.zeros(n)
    (ix, wx), (iy, wy), (iz, wz) = _stencils(pos, h, n, width, radius)
    for i in range(pos.shape[0]):
        w = q[i] * wx[i][:, None, None] * wy[i][None, :, None] * wz[i][None, None, :]
        np.add.at(out, (ix[i][:, None, None], iy[i][None, :, None], iz[i][None, None, :]), w)
    return out


def interpolate(fields, pos, L, n, width, radius):
    """gridops.py:176-192 for a (c, nx, ny, nz) stack."""
    h = [L[a] / n[a] for a in range(3)]
    (ix, wx), (iy, wy), (iz, wz) = _stencils(pos, h, n, width, radius)
    vals = np.zeros((fields.shape[0], pos.shape[0]))
    for i in range(pos.shape[0]):
        w = wx[i][:, None, None] * wy[i][None, :, None] * wz[i][None, None, :]
        fv = fields[:, ix[i][:, None, None], iy[i][None, :, None], iz[i][None, None, :]]
        vals[:, i] = (h[0] * h[1] * h[2]) * np.einsum("xyz,cxyz->c", w, fv)
    return vals


def near_forces(pos, q, L, r_cut, g_w, xi, eps):
    """bd.py:335-355 with an all-pairs search."""
    d = pos[:, None, :] - pos[None, :, :]
    for ax in range(3):
        d[..., ax] -= L[ax] * np.round(d[..., ax] / L[ax])
    r = np.sqrt(np.sum(d * d, axis=-1))
    c1, c2 = kernel_widths(g_w, xi, "avg")
    grad = (d_erf_over_r(r, c1) - d_erf_over_r(r, c2)) / (FOUR_PI * eps)
    coef = np.where(r > 0, -grad / np.where(r > 0, r, 1.0), 0.0)
    keep = (r <= r_cut) & ~np.eye(pos.shape[0], dtype=bool)
    coef = np.where(keep, coef, 0.0)
    return np.einsum("ij,ijc->ic", coef * q[None, :], d)


class TpSolver:
    """bd.py:297-331 planning and forces."""

    def __init__(self, box, n_grid, g_w, eps, delta=5e-4):
        from paper_2101_07088_b200.params import tune_cutoff
        self.box = tuple(float(b) for b in box)
        self.eps, self.g_w = float(eps), float(g_w)
        n_g, factor = ACCURACY[delta]
        h = self.box[0] / n_grid
        self.g_t = factor * h
        self.xi = 0.5 / math.sqrt(self.g_t**2 - g_w**2)
        self.radius = 0.5 * n_g * h
        self.r_cut = tune_cutoff(self.xi, g_w, delta) + (0.5 * n_g / factor) * g_w
        self.n = (n_grid, n_grid, max(int(round(self.box[2] / h)), 4))

    def forces(self, pos, q):
        rho = spread(pos, q, self.box, self.n, self.g_t, self.radius)
        _, e = poisson(rho, self.eps, self.box, with_field=True)
        far = interpolate(e, pos, self.box, self.n, self.g_t, self.radius)
        near = near_forces(pos, q, self.box, self.r_cut, self.g_w, self.xi, self.eps)
        return q[:, None] * (far.T + near)
