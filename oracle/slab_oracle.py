"""TEST INFRASTRUCTURE — numpy/scipy restatement of the reference solve.

This module restates, stage by stage, ``SlabSolver.solve`` of the reference
package ``slabewald`` 0.1.0 (``/root/reference/pkg/src/slabewald/slab.py:
259-394``) so the GPU product can be checked on machines where the reference
is absent (the GPU box).  It is the CHECKER: only tests, ``smoke()`` and the
CPU-baseline leg of ``bench.py`` may call it.  See ``oracle/__init__.py``.

Third-party arithmetic the reference delegates (pinned by what is installed
in this image: numpy 2.3.5, scipy 1.18.1): ``scipy.fft`` (pocketfft) for the
xy FFT and the DCT-I, ``scipy.special.erf`` for the pair kernels,
``scipy.spatial.cKDTree`` for neighbour search.  The same libraries are used
here, so the oracle reproduces the reference to rounding.

Layout: grids are ``[Nx, Ny, Nz]`` (z last) exactly as in the reference so
stage captures can be compared with reference dumps without transposes.
"""

import math
import warnings

import numpy as np
import scipy.fft as sfft
from scipy.spatial import cKDTree
from scipy.special import erf

FOUR_PI = 4.0 * np.pi
TWO_OVER_SQRTPI = 2.0 / np.sqrt(np.pi)
CHUNK = 256                 # charges per vectorised chunk (gridops.py:15)


# ---------------------------------------------------------------------------
# Chebyshev primitives  (reference chebyshev.py)
# ---------------------------------------------------------------------------

def cheb_nodes(n, z0, z1):
    """Ascending second-kind Chebyshev points (chebyshev.py:14-19)."""
    t = np.cos(np.pi * np.arange(n - 1, -1, -1) / (n - 1))
    return 0.5 * (z0 + z1) + 0.5 * (z1 - z0) * t


def cc_weights(n, z0, z1):
    """Clenshaw-Curtis weights for :func:`cheb_nodes` (chebyshev.py:22-43)."""
    deg = n - 1
    theta = np.pi * np.arange(1, deg) / deg
    inner = np.ones(deg - 1)
    if deg % 2 == 0:
        end = 1.0 / (deg**2 - 1)
        for k in range(1, deg // 2):
            inner -= 2.0 * np.cos(2 * k * theta) / (4 * k**2 - 1)
        inner -= np.cos(deg * theta) / (deg**2 - 1)
    else:
        end = 1.0 / deg**2
        for k in range(1, (deg - 1) // 2 + 1):
            inner -= 2.0 * np.cos(2 * k * theta) / (4 * k**2 - 1)
    w = np.concatenate([[end], 2.0 * inner / deg, [end]])
    return 0.5 * (z1 - z0) * w[::-1].copy()


def cheb_coeffs(values):
    """Values at ascending nodes (last axis) -> T_n coefficients
    (chebyshev.py:46-54)."""
    n = values.shape[-1]
    a = sfft.dct(values[..., ::-1], type=1, axis=-1) / (2 * (n - 1))
    a[..., 1:n - 1] *= 2.0
    return a


def cheb_values(coeffs):
    """Inverse of :func:`cheb_coeffs` (chebyshev.py:57-65)."""
    n = coeffs.shape[-1]
    b = np.array(coeffs, copy=True)
    b[..., 1:n - 1] *= 0.5
    return sfft.dct(b, type=1, axis=-1)[..., ::-1]


def cheb_deriv(coeffs, z0, z1):
    """Coefficients of d/dz on [z0, z1] (chebyshev.py:68-79)."""
    n = coeffs.shape[-1]
    b = np.zeros_like(coeffs)
    if n >= 2:
        b[..., n - 2] = 2.0 * (n - 1) * coeffs[..., n - 1]
        for m in range(n - 3, -1, -1):
            b[..., m] = b[..., m + 2] + 2.0 * (m + 1) * coeffs[..., m + 1]
        b[..., 0] *= 0.5
    b *= 2.0 / (z1 - z0)
    return b


def cheb_basis_at(n, z, z0, z1):
    """T_0..T_{n-1} at one z (chebyshev.py:82-95; slab.py:218-222)."""
    x = np.clip(2.0 * (z - z0) / (z1 - z0) - 1.0, -1.0, 1.0)
    return np.cos(np.arange(n) * np.arccos(x))


def wavenumbers(nx, ny, lx, ly):
    """fft-ordered angular wavenumbers (chebyshev.py:98-102)."""
    kx = 2.0 * np.pi * sfft.fftfreq(nx, d=1.0 / nx) / lx
    ky = 2.0 * np.pi * sfft.fftfreq(ny, d=1.0 / ny) / ly
    return kx, ky


# ---------------------------------------------------------------------------
# Gaussian spreading / interpolation  (reference gridops.py:18-133)
# ---------------------------------------------------------------------------

def _axis_uniform(p, h, n, radius):
    """Periodic uniform stencil -> (index, offset, in-support mask)."""
    m = int(np.floor(radius / h + 1e-12))
    cols = np.floor(p / h).astype(np.int64)[:, None] + np.arange(-m, m + 1)
    off = p[:, None] - cols * h
    return cols % n, off, np.abs(off) <= radius + 1e-12 * radius


def _axis_cheb(p, nodes, radius):
    """Chebyshev-axis stencil by bisection (gridops.py:29-39)."""
    first = np.searchsorted(nodes, p - radius, side="left")
    stop = np.searchsorted(nodes, p + radius, side="right")
    span = max(int(np.max(stop - first)), 1) if p.size else 1
    raw = first[:, None] + np.arange(span)
    idx = np.minimum(raw, nodes.size - 1)
    off = p[:, None] - nodes[idx]
    return idx, off, (raw < stop[:, None]) & (np.abs(off) <= radius)


def _gauss(off, mask, width):
    w = np.exp(-0.5 * (off / width) ** 2) / np.sqrt(2.0 * np.pi * width**2)
    return np.where(mask, w, 0.0)


class ChebGrid:
    """Uniform periodic x, y and Chebyshev z grid (gridops.py:47-64)."""

    def __init__(self, Lx, Ly, nx, ny, nz, z0, z1):
        self.Lx, self.Ly = float(Lx), float(Ly)
        self.nx, self.ny, self.nz = int(nx), int(ny), int(nz)
        self.z0, self.z1 = float(z0), float(z1)
        self.hx, self.hy = self.Lx / self.nx, self.Ly / self.ny
        self.x = self.hx * np.arange(self.nx)
        self.y = self.hy * np.arange(self.ny)
        self.z = cheb_nodes(self.nz, z0, z1)
        self.wz = cc_weights(self.nz, z0, z1)

    @property
    def shape(self):
        return (self.nx, self.ny, self.nz)

    def stencils(self, p, width, rxy, rz):
        ix, ox, mx = _axis_uniform(p[:, 0], self.hx, self.nx, rxy)
        iy, oy, my = _axis_uniform(p[:, 1], self.hy, self.ny, rxy)
        iz, oz, mz = _axis_cheb(p[:, 2], self.z, rz)
        return ((ix, _gauss(ox, mx, width)), (iy, _gauss(oy, my, width)),
                (iz, _gauss(oz, mz, width)))

    def _check_z(self, p):
        if np.any((p[:, 2] < self.z0) | (p[:, 2] > self.z1)):
            raise ValueError("point outside the extended z domain")

    def spread(self, pos, q, width, rxy, rz):
        p = np.atleast_2d(np.asarray(pos, dtype=float))
        q = np.atleast_1d(np.asarray(q, dtype=float))
        total = np.zeros(self.nx * self.ny * self.nz)
        if p.shape[0] == 0:
            return total.reshape(self.shape)
        self._check_z(p)
        (ix, wx), (iy, wy), (iz, wz) = self.stencils(p, width, rxy, rz)
        # the reference's chunking (_CHUNK = 256, gridops.py:15,91): one
        # full-grid bincount per 256 sources, which is also its cost profile
        step = CHUNK
        for a in range(0, p.shape[0], step):
            s = slice(a, a + step)
            val = (q[s, None, None, None] * wx[s, :, None, None]
                   * wy[s, None, :, None] * wz[s, None, None, :])
            flat = ((ix[s, :, None, None] * self.ny + iy[s, None, :, None])
                    * self.nz + iz[s, None, None, :])
            flat = np.broadcast_to(flat, val.shape)
            total += np.bincount(flat.ravel(), weights=val.ravel(),
                                 minlength=total.size)
        return total.reshape(self.shape)

    def interpolate(self, fields, pos, width, rxy, rz):
        f = np.asarray(fields)
        one = f.ndim == 3
        fs = f[None] if one else f
        p = np.atleast_2d(np.asarray(pos, dtype=float))
        out = np.zeros((fs.shape[0], p.shape[0]))
        if p.shape[0] == 0:
            return out[0] if one else out
        self._check_z(p)
        (ix, wx), (iy, wy), (iz, wz) = self.stencils(p, width, rxy, rz)
        wzq = wz * self.wz[iz]
        step = CHUNK                                      # gridops.py:15,125
        cell = self.hx * self.hy
        for a in range(0, p.shape[0], step):
            s = slice(a, a + step)
            w = wx[s, :, None, None] * wy[s, None, :, None] * wzq[s, None, None, :]
            g = fs[:, ix[s, :, None, None], iy[s, None, :, None],
                   iz[s, None, None, :]]
            out[:, s] = cell * np.einsum('nxyz,cnxyz->cn', w, g)
        return out[0] if one else out


# ---------------------------------------------------------------------------
# Per-mode Chebyshev BVP  (reference bvp.py)
# ---------------------------------------------------------------------------

def integration_maps(n):
    """Band coefficients of the y'' -> y' and y'' -> y maps (bvp.py:21-54):
    y'_m = e_lo[m] y''_{m-1} + e_hi[m] y''_{m+1},
    y_m  = q_lo[m] y''_{m-2} + q_dg[m] y''_m + q_hi[m] y''_{m+2}, m >= 1."""
    e_lo, e_hi = np.zeros(n), np.zeros(n)
    q_lo, q_dg, q_hi = np.zeros(n), np.zeros(n), np.zeros(n)
    if n > 1:
        e_lo[1], e_hi[1] = 1.0, -0.5
        q_dg[1], q_hi[1] = -0.125, 0.125
    if n > 2:
        e_lo[2], e_hi[2] = 0.25, -0.25
        q_lo[2], q_dg[2], q_hi[2] = 0.25, -1.0 / 6.0, 1.0 / 24.0
    for m in range(3, n):
        e_lo[m] = 0.5 / m
        e_hi[m] = -0.5 / m
        q_lo[m] = 1.0 / (4.0 * m * (m - 1))
        q_dg[m] = -0.5 / (m * m - 1.0)
        q_hi[m] = 1.0 / (4.0 * m * (m + 1))
    return e_lo, e_hi, q_lo, q_dg, q_hi


class BvpBank:
    """Factorised mode BVPs ``y'' - k^2 y = f`` on [z0, z1] with decay
    (Robin) ends, one row per distinct |k| (bvp.py:93-278).

    Unknowns: T_n coefficients of y'' plus the two integration constants;
    after splitting even/odd rows the y'' block is two tridiagonals, closed
    by a 2x2 Schur complement."""

    def __init__(self, nz, z0, z1, kvals):
        self.nz = nz
        self.half = 0.5 * (z1 - z0)
        self.maps = integration_maps(nz)
        e_lo, e_hi, q_lo, q_dg, q_hi = self.maps
        self.sgn = np.where(np.arange(nz) % 2 == 0, 1.0, -1.0)
        self.colsum_one = self._colsums(np.ones(nz))
        self.colsum_sgn = self._colsums(self.sgn)
        kap = np.atleast_1d(np.asarray(kvals, dtype=float)) * self.half
        self.kappa = kap
        k2 = kap[:, None] ** 2
        diag = 1.0 - k2 * q_dg
        sub = -k2 * np.broadcast_to(q_lo, (kap.size, nz))
        sup = -k2 * np.broadcast_to(q_hi, (kap.size, nz))
        self.tri = []
        for par in (0, 1):
            lo, dg, up = sub[:, par::2], diag[:, par::2], sup[:, par::2]
            cp = np.zeros_like(dg)
            inv = np.zeros_like(dg)
            inv[:, 0] = 1.0 / dg[:, 0]
            cp[:, 0] = up[:, 0] * inv[:, 0]
            for j in range(1, dg.shape[1]):
                inv[:, j] = 1.0 / (dg[:, j] - lo[:, j] * cp[:, j - 1])
                if j < dg.shape[1] - 1:
                    cp[:, j] = up[:, j] * inv[:, j]
            self.tri.append((lo, cp, inv))
        # A^{-1} B: B puts -kappa^2 in row 0 (constant y_0) and row 1 (y'_0)
        self.ainvb = []
        for par in (0, 1):
            e = np.zeros((kap.size, self.tri[par][0].shape[1]))
            e[:, 0] = -kap**2
            self.ainvb.append(self._thomas(par, None, e))
        (ue, uq), (ve, vq) = self.colsum_one, self.colsum_sgn
        self.crow = (ue[None, :] + kap[:, None] * uq[None, :],
                     ve[None, :] - kap[:, None] * vq[None, :])
        S = np.empty((kap.size, 2, 2))
        for i in range(2):
            for j in range(2):
                full = np.zeros((kap.size, nz))
                full[:, j::2] = self.ainvb[j]
                S[:, i, j] = np.sum(self.crow[i] * full, axis=1)
        S[:, 0, 0] -= kap
        S[:, 0, 1] -= 1.0 + kap
        S[:, 1, 0] -= -kap
        S[:, 1, 1] -= 1.0 + kap
        det = S[:, 0, 0] * S[:, 1, 1] - S[:, 0, 1] * S[:, 1, 0]
        bad = np.abs(det) * 1e12 < np.abs(S).sum(axis=(1, 2)) ** 2
        if np.any(bad):
            raise np.linalg.LinAlgError(
                "ill-conditioned Schur block for kappa=%r" % kap[bad][:5])
        adj = np.empty_like(S)
        adj[:, 0, 0], adj[:, 1, 1] = S[:, 1, 1], S[:, 0, 0]
        adj[:, 0, 1], adj[:, 1, 0] = -S[:, 0, 1], -S[:, 1, 0]
        self.sinv = adj / det[:, None, None]

    def _colsums(self, w):
        e_lo, e_hi, q_lo, q_dg, q_hi = self.maps
        n = self.nz
        ue, uq = np.zeros(n), np.zeros(n)
        ue[:n - 1] += w[1:] * e_lo[1:]
        ue[1:] += w[:n - 1] * e_hi[:n - 1]
        uq[:n - 2] += w[2:] * q_lo[2:]
        uq += w * q_dg
        uq[2:] += w[:n - 2] * q_hi[:n - 2]
        return ue, uq

    def apply_q(self, ypp):
        _, _, q_lo, q_dg, q_hi = self.maps
        y = ypp * q_dg
        y[..., 2:] += ypp[..., :-2] * q_lo[2:]
        y[..., :-2] += ypp[..., 2:] * q_hi[:-2]
        y[..., 0] = 0.0
        return y

    def apply_e(self, ypp):
        e_lo, e_hi = self.maps[0], self.maps[1]
        yp = np.zeros_like(ypp)
        yp[..., 1:] = ypp[..., :-1] * e_lo[1:]
        yp[..., :-1] += ypp[..., 1:] * e_hi[:-1]
        yp[..., 0] = 0.0
        return yp

    def _thomas(self, par, rows, rhs):
        lo, cp, inv = self.tri[par]
        if rows is not None:
            lo, cp, inv = lo[rows], cp[rows], inv[rows]
        n = rhs.shape[1]
        x = np.zeros(rhs.shape, dtype=np.result_type(rhs, inv))
        x[:, 0] = rhs[:, 0] * inv[:, 0]
        for j in range(1, n):
            x[:, j] = (rhs[:, j] - lo[:, j] * x[:, j - 1]) * inv[:, j]
        for j in range(n - 2, -1, -1):
            x[:, j] -= cp[:, j] * x[:, j + 1]
        return x

    def _descend(self, r1, r2, rows):
        ar = np.zeros(r1.shape, dtype=np.result_type(r1, 1.0))
        for par in (0, 1):
            ar[:, par::2] = self._thomas(par, rows, r1[:, par::2])
        srhs = np.stack([np.sum(self.crow[i][rows] * ar, axis=1)
                         for i in range(2)], axis=1) - r2
        c = np.einsum('mij,mj->mi', self.sinv[rows], srhs)
        for j in range(2):
            ar[:, j::2] -= self.ainvb[j][rows] * c[:, j, None]
        return ar, c

    def _residual(self, fsc, bc, ypp, c, rows):
        kap = self.kappa[rows]
        k2 = kap[:, None] ** 2
        r1 = fsc - (ypp - k2 * self.apply_q(ypp))
        r1[:, 0] += k2[:, 0] * c[:, 0]
        r1[:, 1] += k2[:, 0] * c[:, 1]
        yq, ye = self.apply_q(ypp), self.apply_e(ypp)
        one = np.ones(self.nz)
        cdot = np.stack([ye @ one + kap * (yq @ one),
                         ye @ self.sgn - kap * (yq @ self.sgn)], axis=1)
        ddot = np.stack([kap * c[:, 0] + (1.0 + kap) * c[:, 1],
                         -kap * c[:, 0] + (1.0 + kap) * c[:, 1]], axis=1)
        return r1, bc - (cdot + ddot)

    def solve(self, f, rows, refine=1):
        """f: (M, nz) coefficients of the right-hand side; rows: factor row
        of each batch row.  Returns y coefficients (alpha = beta = 0)."""
        fsc = f * self.half**2
        bc = np.zeros((f.shape[0], 2), dtype=np.result_type(f, 1.0))
        ypp, c = self._descend(fsc, bc, rows)
        for _ in range(refine):
            d1, d2 = self._residual(fsc, bc, ypp, c, rows)
            dy, dc = self._descend(d1, d2, rows)
            ypp += dy
            c += dc
        y = self.apply_q(ypp)
        y[:, 0] += c[:, 0]
        if self.nz > 1:
            y[:, 1] += c[:, 1]
        return y

    def solve_k0(self, f):
        """k = 0: y'' = f, y(z0) = y(z1) = 0 (bvp.py:281-296)."""
        y = self.apply_q(np.asarray(f) * self.half**2)
        top = np.sum(y, axis=-1)
        bot = np.sum(y * self.sgn, axis=-1)
        y[..., 0] += -0.5 * (top + bot)
        if self.nz > 1:
            y[..., 1] += 0.5 * (bot - top)
        return y


class ModeSolver:
    """eps lap psi = -rho per xy mode (dpsolver.py:26-71)."""

    CHUNK = 32768

    def __init__(self, nx, ny, nz, Lx, Ly, z0, z1, eps):
        self.eps = float(eps)
        self.shape = (nx, ny, nz)
        self.kx, self.ky = wavenumbers(nx, ny, Lx, Ly)
        self.kmag = np.hypot(self.kx[:, None], self.ky[None, :])
        flat = self.kmag.ravel()
        self.nonzero = np.flatnonzero(flat > 0.0)
        uniq, self.rows = np.unique(flat[self.nonzero], return_inverse=True)
        self.bank = BvpBank(nz, z0, z1, uniq)

    def solve(self, rho_coeffs, refine=1):
        nx, ny, nz = self.shape
        lead = rho_coeffs.shape[:-3]
        f = -rho_coeffs.reshape((-1, nx * ny, nz)) / self.eps
        out = np.zeros_like(f)
        out[:, 0] = self.bank.solve_k0(f[:, 0])
        ns = f.shape[0]
        step = max(self.CHUNK // ns, 1)
        for a in range(0, self.nonzero.size, step):
            cols = self.nonzero[a:a + step]
            rows = self.rows[a:a + step]
            y = self.bank.solve(f[:, cols].reshape(-1, nz), np.tile(rows, ns),
                                refine)
            out[:, cols] = y.reshape(ns, cols.size, nz)
        return out.reshape(lead + (nx, ny, nz))


def correction_tables(eps, eps_b, eps_t, H, kmag, znodes, z_lo, z_hi, k_max):
    """Harmonic-correction response tables in extended precision
    (dpsolver.py:101-129).  Returns (sel, win, p_b, p_t, d_b, d_t)."""
    sel = (kmag > 0.0) & (kmag <= k_max)
    win = (znodes >= z_lo) & (znodes <= z_hi)
    if not (np.any(sel) and np.any(win)):
        return np.zeros_like(sel), win, None, None, None, None
    ld = np.longdouble
    k = kmag[sel].astype(ld)[:, None]
    z = znodes[win].astype(ld)[None, :]
    rb, rt, Hl = ld(eps_b) / ld(eps), ld(eps_t) / ld(eps), ld(H)
    den = k * ((1 + rb) * (1 + rt) - (1 - rb) * (1 - rt) * np.exp(-2 * k * Hl))
    e1, e2 = np.exp(-k * z), np.exp(k * (z - Hl))
    e3, e4 = np.exp(-k * (Hl + z)), np.exp(k * (z - 2 * Hl))
    p_b = (((rt + 1) * e1 - (rt - 1) * e4) / den).astype(float)
    p_t = ((-(rb + 1) * e2 + (rb - 1) * e3) / den).astype(float)
    d_b = (-k * ((rt + 1) * e1 + (rt - 1) * e4) / den).astype(float)
    d_t = (-k * ((rb + 1) * e2 + (rb - 1) * e3) / den).astype(float)
    return sel, win, p_b, p_t, d_b, d_t


# ---------------------------------------------------------------------------
# Pair kernels  (reference kernels.py)
# ---------------------------------------------------------------------------

def erf_over_r(r, c):
    r = np.asarray(r, dtype=float)
    if np.isinf(c):
        return np.zeros_like(r)
    tiny = r < 1e-10 * c
    rr = np.where(tiny, 1.0, r)
    return np.where(tiny, TWO_OVER_SQRTPI / c, erf(rr / c) / rr)


def d_erf_over_r(r, c):
    r = np.asarray(r, dtype=float)
    if np.isinf(c):
        return np.zeros_like(r)
    tiny = r < 1e-2 * c
    rr = np.where(tiny, c, r)
    x = rr / c
    closed = TWO_OVER_SQRTPI * np.exp(-x * x) / (c * rr) - erf(x) / rr**2
    u = (r / c) ** 2
    series = TWO_OVER_SQRTPI / c**2 * (r / c) * (
        -2.0 / 3.0 + u * (2.0 / 5.0 + u * (-1.0 / 7.0 + u / 27.0)))
    return np.where(tiny, series, closed)


def kernel_widths(g_w, xi, kind):
    """(c1, c2) of the near kernel (erf(r/c1) - erf(r/c2)) / (4 pi eps r)."""
    if kind == "avg":
        c2 = 2.0 * g_w if np.isinf(xi) else np.sqrt(4.0 * g_w**2 + 1.0 / xi**2)
        return 2.0 * g_w, c2
    c2 = np.sqrt(2.0) * g_w if np.isinf(xi) else \
        np.sqrt(2.0 * g_w**2 + 1.0 / xi**2)
    return np.sqrt(2.0) * g_w, c2


def self_avg(g_w, xi, eps, subtract_unsplit=False):
    c2 = kernel_widths(g_w, xi, "avg")[1]
    if subtract_unsplit:
        return -TWO_OVER_SQRTPI / c2 / (FOUR_PI * eps)
    return TWO_OVER_SQRTPI * (0.5 / g_w - 1.0 / c2) / (FOUR_PI * eps)


class NearSources:
    """Charges plus one mirrored layer per jumping wall, periodic-xy
    KD-tree (slab.py:85-181)."""

    def __init__(self, pos, q, geo, par):
        self.geo, self.par = geo, par
        self.empty = pos.shape[0] == 0 or np.isinf(par.xi)
        if self.empty:
            return
        if par.r_cut >= 0.5 * min(geo.Lx, geo.Ly):
            raise ValueError("near-field cutoff exceeds half the periodic box")
        fb = geo.image_strength_bottom(1.0)
        ft = geo.image_strength_top(1.0)
        src, sq = [pos], [q]
        if fb != 0.0:
            m = pos.copy()
            m[:, 2] *= -1.0
            src.append(m)
            sq.append(fb * q)
        if ft != 0.0:
            m = pos.copy()
            m[:, 2] = 2.0 * geo.H - m[:, 2]
            src.append(m)
            sq.append(ft * q)
        self.src = np.concatenate(src, axis=0)
        self.sq = np.concatenate(sq)
        self.zmin = self.src[:, 2].min() - par.r_cut - 1.0
        lz = (self.src[:, 2].max() - self.zmin) + 2.0 * par.r_cut + 2.0
        self.tree = cKDTree(self._shift(self.src),
                            boxsize=np.array([geo.Lx, geo.Ly, lz]))

    def _shift(self, p):
        s = np.empty_like(p)
        s[:, 0] = np.mod(p[:, 0], self.geo.Lx)
        s[:, 1] = np.mod(p[:, 1], self.geo.Ly)
        s[:, 2] = p[:, 2] - self.zmin
        return s

    def pairs(self, ev, radius):
        lists = self.tree.query_ball_point(self._shift(ev), r=radius)
        cnt = np.fromiter((len(l) for l in lists), dtype=np.int64,
                          count=len(lists))
        if cnt.sum() == 0:
            z = np.zeros(0, dtype=np.int64)
            return z, z, np.zeros((0, 3)), np.zeros(0)
        sj = np.concatenate([np.asarray(l, dtype=np.int64) for l in lists
                             if l])
        ti = np.repeat(np.arange(ev.shape[0]), cnt)
        d = ev[ti] - self.src[sj]
        d[:, 0] -= self.geo.Lx * np.round(d[:, 0] / self.geo.Lx)
        d[:, 1] -= self.geo.Ly * np.round(d[:, 1] / self.geo.Ly)
        r = np.sqrt(np.sum(d * d, axis=1))
        keep = r <= radius
        return ti[keep], sj[keep], d[keep], r[keep]

    def evaluate(self, ev, kind="avg", need_field=True, subtract_unsplit=False,
                 chunk=8192):
        ne = ev.shape[0]
        phi = np.zeros(ne)
        efield = np.zeros((ne, 3))
        if self.empty:
            return (phi, efield) if need_field else phi
        par, eps = self.par, self.geo.eps
        c1, c2 = kernel_widths(par.g_w, par.xi, kind)
        radius = par.r_cut if kind == "avg" else par.r_nf
        for a in range(0, ne, chunk):
            ti, sj, d, r = self.pairs(ev[a:a + chunk], radius)
            zero = r == 0.0
            g = (erf_over_r(r, c1) - erf_over_r(r, c2)) / (FOUR_PI * eps)
            if kind == "avg":
                g = np.where(zero, self_avg(par.g_w, par.xi, eps,
                                            subtract_unsplit), g)
            else:
                g0 = (TWO_OVER_SQRTPI / c1 - TWO_OVER_SQRTPI / c2) \
                    / (FOUR_PI * eps)
                g = np.where(zero, g0, g)
            n_here = min(chunk, ne - a)
            phi[a:a + n_here] = np.bincount(ti, weights=self.sq[sj] * g,
                                            minlength=n_here)
            if need_field:
                grad = (d_erf_over_r(r, c1) - d_erf_over_r(r, c2)) \
                    / (FOUR_PI * eps)
                coef = np.where(zero, 0.0, -self.sq[sj] * grad
                                / np.where(zero, 1.0, r))
                for ax in range(3):
                    efield[a:a + n_here, ax] = np.bincount(
                        ti, weights=coef * d[:, ax], minlength=n_here)
        return (phi, efield) if need_field else phi


# ---------------------------------------------------------------------------
# The solve  (reference slab.py:194-461)
# ---------------------------------------------------------------------------

def partition(pos, q, geo, par):
    """C_over / C_far split and first images (slab.py:51-82)."""
    z = pos[:, 2]
    nb = z < 2.0 * par.H_E
    nt = z > geo.H - 2.0 * par.H_E
    over = np.flatnonzero(nb | nt)
    far = np.flatnonzero(~(nb | nt))
    fb = geo.image_strength_bottom(1.0)
    ft = geo.image_strength_top(1.0)
    # per over-charge: bottom image first, then top image (loop order)
    rows = []
    for idx in over:
        if nb[idx] and fb != 0.0:
            rows.append((pos[idx, 0], pos[idx, 1], -pos[idx, 2],
                         fb * q[idx], idx, 0))
        if nt[idx] and ft != 0.0:
            rows.append((pos[idx, 0], pos[idx, 1], 2.0 * geo.H - pos[idx, 2],
                         ft * q[idx], idx, 1))
    if rows:
        arr = np.array(rows, dtype=float)
        ipos, istr = arr[:, :3].copy(), arr[:, 3].copy()
        isrc, iwall = arr[:, 4].astype(int), arr[:, 5].astype(int)
    else:
        ipos, istr = np.zeros((0, 3)), np.zeros(0)
        isrc, iwall = np.zeros(0, dtype=int), np.zeros(0, dtype=int)
    return dict(over=over, far=far, image_positions=ipos,
                image_strengths=istr, image_source=isrc, image_wall=iwall)


class OracleSlabSolver:
    """CPU restatement of ``SlabSolver`` (same constructor / solve API)."""

    def __init__(self, system, params, refine=1, workers=1):
        self.system, self.params = system, params
        self.refine, self.workers = refine, workers
        geo, par = system.geometry, params
        self.grid = ChebGrid(geo.Lx, geo.Ly, par.Nx, par.Ny, par.Nz, par.z0,
                             par.z1)
        self.modes = ModeSolver(par.Nx, par.Ny, par.Nz, geo.Lx, geo.Ly,
                                par.z0, par.z1, geo.eps)
        self.corr = correction_tables(geo.eps, geo.eps_b, geo.eps_t, geo.H,
                                      self.modes.kmag, self.grid.z, -par.H_E,
                                      geo.H + par.H_E, par.k_max)
        self.sigma_b, self.sigma_t = system.surface.sample(geo, par.Nx, par.Ny)
        nxy = par.Nx * par.Ny
        self.sb_hat = sfft.fft2(self.sigma_b) / nxy
        self.st_hat = sfft.fft2(self.sigma_t) / nxy
        self.t_wall = {z: cheb_basis_at(par.Nz, z, par.z0, par.z1)
                       for z in (0.0, geo.H)}
        ikx, iky = 1j * self.modes.kx, 1j * self.modes.ky
        if par.Nx % 2 == 0:
            ikx[par.Nx // 2] = 0.0
        if par.Ny % 2 == 0:
            iky[par.Ny // 2] = 0.0
        self.ikx, self.iky = ikx, iky
        qs = np.abs(system.charges).sum() / geo.area
        ss = np.abs(self.sigma_b).mean() + np.abs(self.sigma_t).mean()
        self.k0_scale = (qs + ss) / geo.eps

    # -- stages --------------------------------------------------------
    def _spread(self, pos, q):
        p = self.params
        return self.grid.spread(pos, q, p.g_t, p.H_E, p.H_E)

    def _forward(self, rho):
        nxy = self.params.Nx * self.params.Ny
        hat = sfft.fft2(rho, axes=(0, 1), workers=self.workers) / nxy
        return cheb_coeffs(hat)

    def _to_grid(self, modes):
        nxy = self.params.Nx * self.params.Ny
        return sfft.ifft2(modes * nxy, axes=(0, 1), workers=self.workers).real

    def _apply_correction(self, mism):
        geo = self.system.geometry
        sel, win, p_b, p_t, d_b, d_t = self.corr
        shape = self.grid.shape
        val = np.zeros(shape, dtype=complex)
        dval = np.zeros(shape, dtype=complex)
        for name, arr in mism.items():
            if not np.all(np.isfinite(arr)):
                raise FloatingPointError("non-finite mismatch field " + name)
        if not np.any(sel):
            return val, dval
        k = self.modes.kmag[sel]
        mb = (mism["e_b"][sel] - geo.eps_b * k * mism["phi_b"][sel]) / geo.eps
        mt = (geo.eps_t * k * mism["phi_t"][sel] + mism["e_t"][sel]) / geo.eps
        tmp = np.zeros((k.size, shape[2]), dtype=complex)
        tmp[:, win] = p_b * mb[:, None] + p_t * mt[:, None]
        val[sel] = tmp
        tmp = np.zeros_like(tmp)
        tmp[:, win] = d_b * mb[:, None] + d_t * mt[:, None]
        dval[sel] = tmp
        return val, dval

    def _k0_jump(self, psi_i, dpsi_i, psi_o, dpsi_o, cb, ct):
        geo, par = self.system.geometry, self.params
        T0, TH = self.t_wall[0.0], self.t_wall[geo.H]
        pi0, dpi0 = psi_i[0, 0].real, dpsi_i[0, 0].real
        po0, dpo0 = psi_o[0, 0].real, dpsi_o[0, 0].real
        sgn = self.modes.bank.sgn
        a_b = -(cb * float(dpo0 @ sgn))
        a_t = -(ct * float(dpo0 @ np.ones(par.Nz)))
        ai1 = (geo.eps_b * (cb * float(dpo0 @ T0) + a_b)
               - geo.eps * float(dpi0 @ T0) - self.sb_hat[0, 0].real) / geo.eps
        ai2 = (geo.eps_t * (ct * float(dpo0 @ TH) + a_t)
               - geo.eps * float(dpi0 @ TH) + self.st_hat[0, 0].real) / geo.eps
        return self._k0_finish(ai1, ai2, a_b, a_t, float(pi0 @ T0),
                               float(pi0 @ TH), cb * float(po0 @ T0),
                               ct * float(po0 @ TH), check=True)

    def _k0_plain(self, psi_i, dpsi_i, s0b=0.0, s0t=0.0):
        geo, par = self.system.geometry, self.params
        dpi0, pi0 = dpsi_i[0, 0].real, psi_i[0, 0].real
        ai1 = -float(dpi0 @ self.modes.bank.sgn) - s0b / geo.eps
        ai2 = -float(dpi0 @ np.ones(par.Nz)) + s0t / geo.eps
        b = float(pi0 @ self.t_wall[0.0])
        t = float(pi0 @ self.t_wall[geo.H])
        return self._k0_finish(ai1, ai2, ai1, ai2, b, t, b, t, check=False)

    def _k0_finish(self, ai1, ai2, a_b, a_t, pib, pit, pbb, ptt, check):
        ref = max(abs(ai1), abs(ai2), abs(self.k0_scale))
        disc = abs(ai1 - ai2) / ref if ref > 0 else 0.0
        if check:
            if disc > 1e-2:
                raise FloatingPointError(
                    "k=0 coefficient mismatch %.2e: system not electroneutral"
                    " or under-resolved" % disc)
            if disc > 1e-3:
                warnings.warn("k=0 coefficient mismatch %.2e" % disc)
        return dict(A_i=0.5 * (ai1 + ai2), A_b=a_b, A_t=a_t, ai1=ai1, ai2=ai2,
                    discrepancy=disc, psi_i_bottom=pib, psi_i_top=pit,
                    psi_b_bottom=pbb, psi_t_top=ptt)

    def interp_gamma(self, field, pts):
        par = self.params
        w = par.screen_width
        rad = (par.H_E / par.g_t) * w
        return self.grid.interpolate(field, pts, w, rad, rad)

    # -- solve ---------------------------------------------------------
    # The solve is written as three phases so a sharded host (charges split
    # by index across ranks, grids summed between phases 1 and 2) can drive
    # it; ``solve`` runs them back to back (reference slab.py:259-394).
    def _two_grids(self, include_correction, force_general):
        geo = self.system.geometry
        jumps = geo.eps_b != geo.eps or geo.eps_t != geo.eps or force_general
        return include_correction and jumps

    def spread_phase(self, pos, q, include_correction=True,
                     force_general=False, cap=None):
        """Grids of the charges ``pos, q`` (slab.py:280-297): stacked
        (rho_over, rho_in) with jumps + correction, else (rho,)."""
        geo, par = self.system.geometry, self.params
        cap = cap if cap is not None else {}
        if self._two_grids(include_correction, force_general):
            part = partition(pos, q, geo, par)
            cap["partition"] = part
            rho_o = self._spread(pos[part["over"]], q[part["over"]])
            xp = np.concatenate([pos[part["far"]], part["image_positions"]])
            xq = np.concatenate([q[part["far"]], part["image_strengths"]])
            rho_i = rho_o + self._spread(xp, xq)
            cap["rho_over"], cap["rho_in"] = rho_o, rho_i
            return np.stack([rho_o, rho_i])
        rho = self._spread(pos, q)
        cap["rho_in"] = rho
        return rho[None]

    def field_phase(self, rho, need_forces=True, include_correction=True,
                    force_general=False, cap=None):
        """Mode solves, correction, k = 0 and the field grids from the
        (summed) grids (slab.py:298-352)."""
        geo, par = self.system.geometry, self.params
        cap = cap if cap is not None else {}
        two = self._two_grids(include_correction, force_general)
        if two:
            both = self.modes.solve(np.stack([self._forward(rho[0]),
                                              self._forward(rho[1])]),
                                    self.refine)
            psi_o, psi_i = both[0], both[1]
        else:
            psi_o = None
            psi_i = self.modes.solve(self._forward(rho[0]), self.refine)
        cap["psi_i"], cap["psi_o"] = psi_i, psi_o
        dpsi_i = cheb_deriv(psi_i, par.z0, par.z1)

        T0, TH = self.t_wall[0.0], self.t_wall[geo.H]
        if two:
            dpsi_o = cheb_deriv(psi_o, par.z0, par.z1)
            cb, ct = geo.exterior_factor_bottom(), geo.exterior_factor_top()
            mism = {
                "phi_b": psi_i @ T0 - cb * (psi_o @ T0),
                "e_b": geo.eps * (dpsi_i @ T0)
                - geo.eps_b * cb * (dpsi_o @ T0) + self.sb_hat,
                "phi_t": psi_i @ TH - ct * (psi_o @ TH),
                "e_t": geo.eps * (dpsi_i @ TH)
                - geo.eps_t * ct * (dpsi_o @ TH) - self.st_hat,
            }
            corr, dcorr = self._apply_correction(mism)
            k0 = self._k0_jump(psi_i, dpsi_i, psi_o, dpsi_o, cb, ct)
        elif include_correction:
            zero = np.zeros_like(self.sb_hat)
            mism = {"phi_b": zero, "e_b": self.sb_hat, "phi_t": zero,
                    "e_t": -self.st_hat}
            corr, dcorr = self._apply_correction(mism)
            k0 = self._k0_plain(psi_i, dpsi_i, self.sb_hat[0, 0].real,
                                self.st_hat[0, 0].real)
        else:
            mism = None
            corr = dcorr = None
            k0 = self._k0_plain(psi_i, dpsi_i)
        cap["mismatch"], cap["k0"] = mism, k0
        cap["corr"], cap["dcorr"] = corr, dcorr

        vals = cheb_values(psi_i)
        if corr is not None:
            vals = vals + corr
        psi_vals = self._to_grid(vals) + k0["A_i"] * self.grid.z[None, None, :]
        fields = [psi_vals]
        if need_forces:
            dz = cheb_values(dpsi_i)
            if dcorr is not None:
                dz = dz + dcorr
            fields.append(-self._to_grid(vals * self.ikx[:, None, None]))
            fields.append(-self._to_grid(vals * self.iky[None, :, None]))
            fields.append(-(self._to_grid(dz) + k0["A_i"]))
        stack = np.stack(fields)
        cap["fields"] = stack
        return {"k0": k0, "psi_vals": psi_vals, "fields": stack}

    def charge_phase(self, state, pos, q, first=0, count=None,
                     need_energy=True, need_forces=True, need_potential=True,
                     subtract_self=False, cap=None, near_ext=None, near0_ext=None):
        """Interpolation, near field, gauge and energy at the charges
        ``first .. first+count-1`` with every charge as a near-field source
        (slab.py:354-391).  Returns (phi, E, U_part, diag); the parts of U
        over a partition of the charges sum to U (the wall-charge energy is
        added by the part holding charge 0)."""
        geo, par = self.system.geometry, self.params
        cap = cap if cap is not None else {}
        n = pos.shape[0]
        count = n - first if count is None else count
        own = slice(first, first + count)
        k0, psi_vals, stack = state["k0"], state["psi_vals"], state["fields"]
        pe, qe = pos[own], q[own]
        far = self.grid.interpolate(stack, pe, par.g_t, par.H_E, par.H_E)
        nf = NearSources(pos, q, geo, par) if near_ext is None else None
        if near_ext is not None:
            # near-field sums supplied by the caller (the cell-routed sharded
            # solve computes them on the rank owning each charge's cell)
            phi_near = near_ext[0]
            e_near = np.stack(near_ext[1:4], axis=1) if need_forces else None
            e_bar = far[1:4].T + e_near if need_forces else np.zeros((pe.shape[0], 3))
        elif need_forces:
            phi_near, e_near = nf.evaluate(pe, "avg",
                                           subtract_unsplit=subtract_self)
            e_bar = far[1:4].T + e_near
        else:
            phi_near = nf.evaluate(pe, "avg", need_field=False,
                                   subtract_unsplit=subtract_self)
            e_near = None
            e_bar = np.zeros((pe.shape[0], 3))
        cap["phi_far"], cap["phi_near"], cap["e_near"] = far[0], phi_near, e_near
        if subtract_self and np.isinf(par.xi):
            phi_near = phi_near + qe * self_avg(par.g_w, np.inf, geo.eps, True)
        phi_bar = far[0] + phi_near

        b_i = 0.0
        if need_potential and not np.isinf(par.xi):
            origin = np.zeros((1, 3))
            far0 = self.interp_gamma(psi_vals, origin)[0]
            near0 = near0_ext if near_ext is not None else \
                nf.evaluate(origin, "point", need_field=False)[0]
            b_i = -(far0 + near0)
            phi_bar = phi_bar + b_i

        U = 0.0
        if need_energy:
            U = 0.5 * float(np.dot(qe, phi_bar))
            if not self.system.surface.is_zero and first == 0:
                U += self._wall_energy(nf, psi_vals, b_i)
        diag = {"charges": q, "ai1": k0["ai1"], "ai2": k0["ai2"],
                "ai_discrepancy": k0["discrepancy"], "B_i": b_i, "k0": k0,
                "constraints": par.constraints}
        return phi_bar, e_bar, U, diag

    def solve(self, positions=None, need_energy=True, need_forces=True,
              need_potential=True, subtract_self=False,
              include_correction=True, force_general=False, capture=None):
        pos = self.system.positions if positions is None else \
            np.atleast_2d(np.asarray(positions, dtype=float))
        q = self.system.charges
        cap = capture if capture is not None else {}
        rho = self.spread_phase(pos, q, include_correction, force_general, cap)
        state = self.field_phase(rho, need_forces, include_correction,
                                 force_general, cap)
        return self.charge_phase(state, pos, q, 0, pos.shape[0], need_energy,
                                 need_forces, need_potential, subtract_self,
                                 cap)

    def _wall_energy(self, nf, psi_vals, b_i):
        geo = self.system.geometry
        xg, yg = np.meshgrid(self.grid.x, self.grid.y, indexing="ij")
        total = 0.0
        for sigma, z in ((self.sigma_b, 0.0), (self.sigma_t, geo.H)):
            pts = np.column_stack([xg.ravel(), yg.ravel(),
                                   np.full(xg.size, z)])
            phi_w = self.interp_gamma(psi_vals, pts) \
                + nf.evaluate(pts, "point", need_field=False) + b_i
            total += 0.5 * self.grid.hx * self.grid.hy * float(
                sigma.ravel() @ phi_w)
        return total


def oracle_solve(system, params, **kw):
    """One-shot oracle solve -> (phi_bar, E_bar, U, diagnostics)."""
    refine = kw.pop("refine", 1)
    return OracleSlabSolver(system, params, refine=refine).solve(**kw)
