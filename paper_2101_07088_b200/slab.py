"""Drop-in ``SlabSolver`` running on a B200.

Mirrors the reference solver API (``slabewald/slab.py``): ``SlabSolver(
system, params, threads=1, refine=1)``, ``.solve(...)`` with the same
keyword flags, ``SolveResult`` with the same diagnostics keys, plus
``build_partition``, ``near_field_sum`` and ``solve_system``.  Every solve
runs on the GPU through ``libslabewald_cuda.so`` (include/slabewald.h); there
is no CPU fallback.  ``threads`` is accepted for signature compatibility and
ignored (the reference uses it for scipy.fft workers).
"""

import ctypes
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .chebgrid import GridInfo, basis_at, wavenumbers
from .kernels import self_potential_avg


@dataclass
class ChargePartition:
    """Near-wall charges, mid-slab charges and first-layer images
    (reference slab.py:27-36)."""

    over: np.ndarray
    far: np.ndarray
    image_positions: np.ndarray
    image_strengths: np.ndarray
    image_source: np.ndarray
    image_wall: np.ndarray


@dataclass
class K0Coefficients:
    """Linear modes of the k = 0 component (reference dpsolver.py:166-186)."""

    A_i: float
    A_b: float
    A_t: float
    ai1: float
    ai2: float
    discrepancy: float
    psi_i_bottom: float
    psi_i_top: float
    psi_b_bottom: float
    psi_t_top: float

    def offsets_given_Bi(self, B_i, H):
        B_b = self.psi_i_bottom + B_i - self.psi_b_bottom
        B_t = (self.psi_i_top - self.psi_t_top
               + (self.A_i - self.A_t) * H + B_i)
        return B_b, B_t


@dataclass
class SolveResult:
    phi_bar: np.ndarray
    E_bar: np.ndarray
    U: float
    diagnostics: dict = field(default_factory=dict)

    @property
    def forces(self):
        return self.diagnostics["charges"][:, None] * self.E_bar


def _flags(need_energy, need_forces, need_potential, subtract_self,
           include_correction, force_general, timings=False, fp32=False,
           record_pairs=False, graph=False):
    f = 0
    if graph:
        f |= _lib.GRAPH
    if record_pairs:
        f |= _lib.PAIR_HASH
    if fp32:
        f |= _lib.FP32
    if need_energy:
        f |= _lib.NEED_ENERGY
    if need_forces:
        f |= _lib.NEED_FORCES
    if need_potential:
        f |= _lib.NEED_POTENTIAL
    if subtract_self:
        f |= _lib.SUBTRACT_SELF
    if include_correction:
        f |= _lib.CORRECTION
    if force_general:
        f |= _lib.FORCE_GENERAL
    if timings:
        f |= _lib.TIMINGS
    return f


STAGES = ("sources", "spread", "forward", "bvp", "inverse", "interp", "near",
          "finish", "k_spread", "k_bvp", "k_interp", "k_near", "k_near_scan",
          "k_near_eval")


PRECISIONS = ("fp64", "fp32")


def _host_outputs(n, need_forces):
    """Fresh phi (n,) and E (n, 3) arrays in page-locked memory (torch's
    caching host allocator, returned to its pool when the arrays are
    dropped), so the device->host copies run at full link speed."""
    try:
        import torch
        phi = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
        E = torch.empty((n, 3), dtype=torch.float64, pin_memory=True).numpy()
        if not need_forces:
            E[...] = 0.0
        return phi, E
    except (ImportError, RuntimeError):
        return np.empty(n), np.zeros((n, 3))


class SlabSolver:
    """Reusable GPU solver: grids, BVP factorisations and wall data live in
    a device plan created here (reference slab.py:194-233).

    ``precision="fp32"`` (not in the reference) evaluates the near-field pair
    kernels in single precision; pair membership stays the exact fp64 test
    and the results stay within the run's Ewald tolerance."""

    def __init__(self, system, params, threads=1, refine=1, device=0,
                 precision="fp64"):
        if precision not in PRECISIONS:
            raise ValueError("precision must be one of %s" % (PRECISIONS,))
        self.precision = precision
        self.system = system
        self.params = params
        self.threads = threads
        self.refine = refine
        self.device = device
        self._lib = _lib.load()
        geo = system.geometry
        par = params
        self.grid = GridInfo(geo.Lx, geo.Ly, par.Nx, par.Ny, par.Nz, par.z0,
                             par.z1)
        kx, ky = wavenumbers(par.Nx, par.Ny, geo.Lx, geo.Ly)
        t0 = basis_at(par.Nz, 0.0, par.z0, par.z1)
        tH = basis_at(par.Nz, geo.H, par.z0, par.z1)
        self.sigma_b, self.sigma_t = system.surface.sample(geo, par.Nx, par.Ny)
        sb = st = None
        if not system.surface.is_zero:
            sb = _lib.as_f64(self.sigma_b)
            st = _lib.as_f64(self.sigma_t)
        self._consts = [_lib.as_f64(a) for a in (self.grid.z, self.grid.wz,
                                                 t0, tH, kx, ky)]
        self._pstruct = _lib.params_struct(geo, par, refine)
        handle = ctypes.c_void_p()
        z, wz, t0c, tHc, kxc, kyc = self._consts
        _lib.check(self._lib.se_plan_create(
            ctypes.byref(self._pstruct), _lib.dptr(z), _lib.dptr(wz),
            _lib.dptr(t0c), _lib.dptr(tHc), _lib.dptr(kxc), _lib.dptr(kyc),
            _lib.dptr(sb), _lib.dptr(st), int(device), ctypes.byref(handle)))
        self._plan = handle
        q = _lib.as_f64(system.charges)
        self._q = q
        _lib.check(self._lib.se_set_charges(self._plan, _lib.dptr(q), q.size))
        self.last_timings = None

    def close(self):
        if getattr(self, "_plan", None):
            self._lib.se_plan_destroy(self._plan)
            self._plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _positions(self, positions):
        if positions is None:
            pos = self.system.positions
        else:
            pos = np.atleast_2d(np.asarray(positions, dtype=float))
        pos = _lib.as_f64(pos)
        if pos.ndim != 2 or (pos.size and pos.shape[1] != 3):
            raise ValueError("positions must be (N, 3)")
        if pos.shape[0] != self._q.size:
            raise ValueError("positions and charges disagree on N")
        return pos.reshape(-1, 3)

    def _diagnostics(self, d):
        q = self.system.charges
        k0 = K0Coefficients(A_i=d.A_i, A_b=d.A_b, A_t=d.A_t, ai1=d.ai1,
                            ai2=d.ai2, discrepancy=d.discrepancy,
                            psi_i_bottom=d.psi_i_bottom,
                            psi_i_top=d.psi_i_top,
                            psi_b_bottom=d.psi_b_bottom,
                            psi_t_top=d.psi_t_top)
        if d.warn_discrepancy:
            warnings.warn("k=0 coefficient mismatch %.2e" % d.discrepancy)
        return {"charges": q, "ai1": d.ai1, "ai2": d.ai2,
                "ai_discrepancy": d.discrepancy, "B_i": d.B_i, "k0": k0,
                "constraints": self.params.constraints,
                "n_sources": int(d.n_sources), "n_pairs": int(d.n_pairs),
                "n_launches": int(d.n_launches)}

    def solve(self, positions=None, need_energy=True, need_forces=True,
              need_potential=True, subtract_self=False,
              include_correction=True, force_general=False, timings=False,
              record_pairs=False, graph=True):
        """Averaged potential and field at every charge, and the energy
        (reference slab.py:259-394).  ``record_pairs`` (not in the reference)
        keeps the near-field pair set for :meth:`pair_set`; ``graph`` (not in
        the reference) replays repeated solves with the same flags as one
        CUDA graph (the positions are copied into the plan's own device
        buffer, so every call reuses the captured solve)."""
        pos = self._positions(positions)
        n = pos.shape[0]
        flags = _flags(need_energy, need_forces, need_potential,
                       subtract_self, include_correction, force_general,
                       timings, self.precision == "fp32", record_pairs,
                       graph=graph)
        phi, E = _host_outputs(n, need_forces)
        U = ctypes.c_double(0.0)
        diag = _lib.SeDiag()
        _lib.check(self._lib.se_solve(
            self._plan, _lib.dptr(pos), n, flags, _lib.dptr(phi),
            _lib.dptr(E) if need_forces else None, ctypes.byref(U),
            ctypes.byref(diag)))
        out = self._diagnostics(diag)
        if timings:
            self.last_timings = dict(zip(STAGES, list(diag.t_ms)[:len(STAGES)]))
            out["timings_ms"] = self.last_timings
        return SolveResult(phi_bar=phi, E_bar=E, U=float(U.value),
                           diagnostics=out)

    def solve_device(self, d_pos, d_phi, d_E, n, need_energy=True,
                     need_forces=True, need_potential=True,
                     subtract_self=False, include_correction=True,
                     force_general=False, timings=False, graph=False):
        """Device-resident variant: ``d_pos``, ``d_phi``, ``d_E`` are raw
        device pointers (ints) on the plan's device.  Returns (U, diag).
        ``graph``: capture the solve as a CUDA graph on the second call with
        the same buffers and flags and replay it from then on."""
        flags = _flags(need_energy, need_forces, need_potential,
                       subtract_self, include_correction, force_general,
                       timings, self.precision == "fp32", graph=graph)
        U = ctypes.c_double(0.0)
        diag = _lib.SeDiag()
        _lib.check(self._lib.se_solve_device(
            self._plan, ctypes.c_void_p(d_pos), int(n), flags,
            ctypes.c_void_p(d_phi), ctypes.c_void_p(d_E), ctypes.byref(U),
            ctypes.byref(diag)))
        if timings:
            self.last_timings = dict(zip(STAGES, list(diag.t_ms)[:len(STAGES)]))
        return float(U.value), diag

    def set_stream(self, stream_handle):
        """Run on a caller's cudaStream_t (int handle, e.g. torch's
        ``torch.cuda.current_stream().cuda_stream``)."""
        _lib.check(self._lib.se_plan_set_stream(self._plan,
                                                ctypes.c_void_p(stream_handle)))

    def pair_set(self):
        """(count[N], hash[N]) of the near-field pairs of the last solve run
        with ``record_pairs=True``: per charge the number of its sources
        within r_cut and the wrap-around sum of splitmix64(source index),
        sources numbered as the reference's NearField (charges, bottom
        mirror layer, top mirror layer; slab.py:104-119)."""
        size = self._lib.se_debug_fetch(self._plan, 6, None, 0)
        if size <= 0:
            raise RuntimeError("no pair set recorded (solve with record_pairs=True)")
        buf = np.empty(size // 8, dtype=np.uint64)
        got = self._lib.se_debug_fetch(self._plan, 6,
                                       buf.ctypes.data_as(ctypes.c_void_p), size)
        if got != size:
            raise RuntimeError("pair set copy failed")
        n = buf.size // 2
        return buf[n:].astype(np.int64), buf[:n].copy()

    def debug_fetch(self, which):
        """Copy a stage buffer of the last solve (see se_debug_fetch)."""
        size = self._lib.se_debug_fetch(self._plan, int(which), None, 0)
        if size < 0:
            raise ValueError("unknown stage buffer %r" % which)
        buf = np.empty(size // 8)
        got = self._lib.se_debug_fetch(self._plan, int(which),
                                       buf.ctypes.data_as(ctypes.c_void_p),
                                       size)
        if got != size:
            raise RuntimeError("stage buffer copy failed")
        return buf


def build_partition(positions, charges, geometry, params):
    """Split charges by wall distance and build their first images
    (reference slab.py:51-82), computed on the device."""
    lib = _lib.load()
    pos = _lib.as_f64(np.atleast_2d(positions)).reshape(-1, 3)
    q = _lib.as_f64(charges).reshape(-1)
    n = pos.shape[0]
    ps = _lib.params_struct(geometry, params)
    over = np.empty(max(n, 1), dtype=np.int64)
    far = np.empty(max(n, 1), dtype=np.int64)
    ipos = np.empty((max(2 * n, 1), 3))
    istr = np.empty(max(2 * n, 1))
    isrc = np.empty(max(2 * n, 1), dtype=np.int64)
    iwall = np.empty(max(2 * n, 1), dtype=np.int32)
    cnt = [ctypes.c_int64(0) for _ in range(3)]
    i64 = ctypes.POINTER(ctypes.c_int64)
    _lib.check(lib.se_build_partition(
        ctypes.byref(ps), 0, _lib.dptr(pos), _lib.dptr(q), n,
        ctypes.byref(cnt[0]), over.ctypes.data_as(i64), ctypes.byref(cnt[1]),
        far.ctypes.data_as(i64), ctypes.byref(cnt[2]), _lib.dptr(ipos),
        _lib.dptr(istr), isrc.ctypes.data_as(i64),
        iwall.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))))
    no, nf, ni = (c.value for c in cnt)
    return ChargePartition(over[:no].copy(), far[:nf].copy(),
                           ipos[:ni].copy(), istr[:ni].copy(),
                           isrc[:ni].astype(int), iwall[:ni].astype(int))


def near_field_sum(positions, charges, geometry, params, eval_positions=None,
                   kernel="avg", need_field=True, subtract_unsplit_self=False,
                   **deprecated):
    """Near-field pair sums on the device (reference slab.py:184-191, same
    signature: ``kernel`` is "avg" (r_cut) or "point" (r_nf)).  The earlier
    keyword ``kind`` is accepted as an alias."""
    if deprecated:
        if set(deprecated) != {"kind"}:
            raise TypeError("near_field_sum() got unexpected keyword(s) %s"
                            % sorted(set(deprecated) - {"kind"}))
        kernel = deprecated["kind"]
    if kernel not in ("avg", "point"):
        raise ValueError("kernel must be 'avg' or 'point'")
    lib = _lib.load()
    pos = _lib.as_f64(np.atleast_2d(positions)).reshape(-1, 3)
    q = _lib.as_f64(charges).reshape(-1)
    ev = pos if eval_positions is None else \
        _lib.as_f64(np.atleast_2d(eval_positions)).reshape(-1, 3)
    ne = ev.shape[0]
    phi = np.zeros(ne)
    E = np.zeros((ne, 3))
    ps = _lib.params_struct(geometry, params)
    _lib.check(lib.se_near_field(
        ctypes.byref(ps), 0, _lib.dptr(pos), _lib.dptr(q), pos.shape[0],
        _lib.dptr(ev), ne, 0 if kernel == "avg" else 1, 1 if need_field else 0,
        1 if subtract_unsplit_self else 0, _lib.dptr(phi),
        _lib.dptr(E) if need_field else None))
    return (phi, E) if need_field else phi


def solve_system(system, params, **kw):
    """One-shot convenience wrapper around :class:`SlabSolver`."""
    solver = SlabSolver(system, params)
    try:
        return solver.solve(**kw)
    finally:
        solver.close()


__all__ = ["ChargePartition", "K0Coefficients", "SolveResult", "SlabSolver",
           "build_partition", "near_field_sum", "solve_system",
           "self_potential_avg"]
