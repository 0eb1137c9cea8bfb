"""Triply periodic twin of the slab solver on the GPU (SURVEY.md section 8f,
next #3).

Mirrors ``slabewald.solve_triply_periodic`` (dpsolver.py:221-249) and
``slabewald.bd.TriplyPeriodicSolver`` (bd.py:297-355): same names, arguments,
planning arithmetic and results; the spread, FFT Poisson solve,
interpolation and near field run in ``libslabewald_cuda.so`` (se_tp_*).
There is no CPU fallback.
"""

import ctypes
import math

import numpy as np

from . import _lib
from .params import ACCURACY_PROFILES, tune_cutoff


class _TpPlan:
    """Owner of one se_tp plan (grid, FFT plans and scratch on the device)."""

    def __init__(self, box, n, eps, device=0):
        self._lib = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(self._lib.se_tp_create(int(device), float(box[0]), float(box[1]),
                                          float(box[2]), int(n[0]), int(n[1]), int(n[2]),
                                          float(eps), ctypes.byref(h)))
        self._h = h
        self.n = tuple(int(v) for v in n)

    def close(self):
        if self._h is not None and self._h.value:
            self._lib.se_tp_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_triply_periodic(rho, eps, Lx, Ly, Lz, with_field=False, workers=1):
    """FFT Poisson solve eps lap(phi) = -rho on a periodic box; the k = 0
    mode of phi is zero.  With ``with_field`` also E = -grad phi as a
    (3, nx, ny, nz) array.  ``workers`` is accepted and ignored."""
    del workers
    rho = _lib.as_f64(rho)
    if rho.ndim != 3:
        raise ValueError("rho must be a 3-d grid")
    plan = _TpPlan((Lx, Ly, Lz), rho.shape, eps)
    try:
        phi = np.empty_like(rho)
        e = np.empty((3,) + rho.shape) if with_field else None
        _lib.check(plan._lib.se_tp_poisson(plan._h, _lib.dptr(rho), 1 if with_field else 0,
                                           _lib.dptr(phi), _lib.dptr(e)))
    finally:
        plan.close()
    return (phi, e) if with_field else phi


class TriplyPeriodicSolver:
    """Split Ewald electrostatics in a periodic box, for BD validation:
    Gaussian spreading on a uniform grid, FFT Poisson solve, pair near field
    under full minimum image (bd.py:297-355)."""

    def __init__(self, box, n_grid, g_w, eps, delta=5e-4, threads=1, device=0):
        self.box = tuple(float(b) for b in box)
        self.eps = float(eps)
        self.g_w = float(g_w)
        n_g, factor = ACCURACY_PROFILES[delta]
        h = self.box[0] / n_grid
        self.g_t = factor * h
        if self.g_t <= g_w:
            raise ValueError("grid too fine for splitting at this g_w")
        self.xi = 0.5 / math.sqrt(self.g_t**2 - g_w**2)
        self.radius = 0.5 * n_g * h
        self.r_cut = tune_cutoff(self.xi, g_w, delta) \
            + (0.5 * n_g / factor) * g_w
        if self.r_cut >= 0.5 * min(self.box):
            raise ValueError("near-field cutoff exceeds half the box")
        self.n = (int(n_grid), int(n_grid), max(int(round(self.box[2] / h)), 4))
        self.threads = threads
        self.device = device
        self._plan = _TpPlan(self.box, self.n, self.eps, device)

    def forces(self, positions, charges):
        """Electrostatic force (q times averaged field) on each charge."""
        pos = _lib.as_f64(np.atleast_2d(positions)).reshape(-1, 3)
        q = _lib.as_f64(np.atleast_1d(charges))
        if q.shape[0] != pos.shape[0]:
            raise ValueError("positions and charges disagree on N")
        out = np.empty_like(pos)
        _lib.check(self._plan._lib.se_tp_forces(
            self._plan._h, _lib.dptr(pos), _lib.dptr(q), pos.shape[0], self.g_t,
            self.radius, self.g_w, self.xi, self.r_cut, _lib.dptr(out)))
        return out

    def forces_device(self, d_pos, d_q, n, d_out, graph=False):
        """Same on device buffers (pointers, e.g. ``tensor.data_ptr()``), on
        the plan's stream (``set_stream``).  ``graph``: capture the kernels as
        a CUDA graph on the second call with the same buffers and replay it
        from then on."""
        if graph != getattr(self, "_graph", False):
            _lib.check(self._plan._lib.se_tp_set_graph(self._plan._h, 1 if graph else 0))
            self._graph = graph
        _lib.check(self._plan._lib.se_tp_forces_device(
            self._plan._h, ctypes.c_void_p(d_pos), ctypes.c_void_p(d_q), int(n), self.g_t,
            self.radius, self.g_w, self.xi, self.r_cut, ctypes.c_void_p(d_out)))

    def set_stream(self, stream):
        _lib.check(self._plan._lib.se_tp_set_stream(self._plan._h, ctypes.c_void_p(stream)))

    def close(self):
        self._plan.close()


__all__ = ["solve_triply_periodic", "TriplyPeriodicSolver"]
