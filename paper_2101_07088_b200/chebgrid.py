"""Host-side grid constants uploaded to the device plan.

Computed once per solver with numpy in the reference's operation order so
the device sees bit-identical Chebyshev nodes, quadrature weights, wall
basis values and wavenumbers (reference chebyshev.py:14-43,98-102 and
slab.py:214-222).  Stencil membership on the device compares particle
coordinates against these nodes, so bit identity matters here.
"""

import numpy as np
import scipy.fft as sfft


def cheb_nodes(n, z0=-1.0, z1=1.0):
    """Second-kind Chebyshev points on [z0, z1], ascending."""
    if n < 2:
        raise ValueError("need at least 2 Chebyshev points")
    x = np.cos(np.pi * np.arange(n - 1, -1, -1) / (n - 1))
    return 0.5 * (z0 + z1) + 0.5 * (z1 - z0) * x


def clenshaw_curtis_weights(n, z0=-1.0, z1=1.0):
    """Clenshaw-Curtis weights matching :func:`cheb_nodes` (ascending)."""
    deg = n - 1
    ang = np.pi * np.arange(1, deg) / deg
    body = np.ones(deg - 1)
    if deg % 2:
        ends = 1.0 / deg**2
        for k in range(1, (deg - 1) // 2 + 1):
            body -= 2.0 * np.cos(2 * k * ang) / (4 * k**2 - 1)
    else:
        ends = 1.0 / (deg**2 - 1)
        for k in range(1, deg // 2):
            body -= 2.0 * np.cos(2 * k * ang) / (4 * k**2 - 1)
        body -= np.cos(deg * ang) / (deg**2 - 1)
    w = np.empty(n)
    w[0] = w[-1] = ends
    w[1:-1] = 2.0 * body / deg
    return 0.5 * (z1 - z0) * w[::-1].copy()


def basis_at(n, z, z0, z1):
    """T_0..T_{n-1} evaluated at a single z in [z0, z1]."""
    theta = np.arccos(np.clip(2.0 * (z - z0) / (z1 - z0) - 1.0, -1.0, 1.0))
    return np.cos(np.arange(n) * theta)


def wavenumbers(nx, ny, lx, ly):
    kx = 2.0 * np.pi * sfft.fftfreq(nx, d=1.0 / nx) / lx
    ky = 2.0 * np.pi * sfft.fftfreq(ny, d=1.0 / ny) / ly
    return kx, ky


class GridInfo:
    """Read-only description of the solver grid (the reference exposes the
    same attributes on ``SlabSolver.grid``)."""

    def __init__(self, Lx, Ly, nx, ny, nz, z0, z1):
        self.Lx, self.Ly = float(Lx), float(Ly)
        self.nx, self.ny, self.nz = int(nx), int(ny), int(nz)
        self.z0, self.z1 = float(z0), float(z1)
        self.hx = self.Lx / self.nx
        self.hy = self.Ly / self.ny
        self.x = self.hx * np.arange(self.nx)
        self.y = self.hy * np.arange(self.ny)
        self.z = cheb_nodes(self.nz, z0, z1)
        self.wz = clenshaw_curtis_weights(self.nz, z0, z1)

    def shape(self):
        return (self.nx, self.ny, self.nz)
