"""Brownian dynamics on top of the B200 solver.

Mirrors the reference module ``slabewald.bd`` (bd.py) for the parts the BD
driver needs (``cmd_bd``, cli.py:174-230): the steric model (bd.py:27-74),
the two-step-noise Euler-Maruyama step with z-bound rejection and xy wrap
(bd.py:77-133), the pairwise steric forces (bd.py:246-270, on the GPU through
``se_steric_forces``) and the mirror-wall forces (bd.py:273-279).  The noise
stream is numpy's Philox generator seeded like the reference, so trajectories
match the reference draw for draw.  ``TriplyPeriodicSolver`` (bd.py:297)
lives in :mod:`.periodic`; the observables / theory curves are out of scope.
"""

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass(frozen=True)
class StericParams:
    """Truncated, mollified repulsion 4 U0 ((2a/r)^2p - (2a/r)^p) + U0, zero
    beyond its minimum at r = 2^(1/p) 2a, force capped below r_m."""

    a: float
    U0: float = 1.0
    r_m: float = 0.0
    p: int = 6

    @property
    def cutoff(self):
        return 2.0 ** (1.0 / self.p) * 2.0 * self.a


def lj_force(r, s):
    """-dU/dr of the uncut 2p-p potential."""
    x = (2.0 * s.a / r) ** s.p
    return 4.0 * s.U0 * s.p * x * (2.0 * x - 1.0) / r


def _core(r, s):
    floor = s.r_m if s.r_m > 0 else 1e-12 * s.a
    return np.maximum(r, floor)


def steric_force(r, s):
    """Capped core, repulsive flank, zero past the cutoff (bd.py:52-57)."""
    r = np.asarray(r, dtype=float)
    return np.where(r > s.cutoff, 0.0, lj_force(_core(r, s), s))


def steric_energy(r, s):
    """Potential matching :func:`steric_force`, zero at the cutoff and
    continued linearly inside r_m (bd.py:60-68)."""
    r = np.asarray(r, dtype=float)
    rc = _core(r, s)
    x = (2.0 * s.a / rc) ** s.p
    u = 4.0 * s.U0 * (x * x - x) + s.U0
    if s.r_m > 0:
        u = u + lj_force(s.r_m, s) * np.maximum(s.r_m - r, 0.0)
    return np.where(r > s.cutoff, 0.0, u)


@dataclass
class BdConfig:
    dt: float
    steps: int
    equil_steps: int = 0
    mu: float = 1.0
    kT: float = 1.0
    seed: int = 0
    max_disp: float = np.inf
    max_retries: int = 100
    sample_every: int = 50


@dataclass
class BdState:
    positions: np.ndarray
    prev_noise: np.ndarray
    rng: np.random.Generator
    rejections: int = 0
    steps_done: int = 0


@dataclass
class Observables:
    """Density (and pair-correlation) histograms with the reference's
    normalisation (bd.py:139-181); host numpy, sampled rarely."""

    H: float
    area: float
    z_bin: float
    r_max: float = 0.0
    r_bin: float = 0.0
    samples: int = 0
    z_counts: np.ndarray = None
    pair_counts: np.ndarray = None
    _pair_norm: float = 0.0

    def __post_init__(self):
        self.z_edges = np.arange(0.0, self.H + self.z_bin, self.z_bin)
        self.z_counts = np.zeros(self.z_edges.size - 1)
        if self.r_max > 0:
            self.r_edges = np.arange(0.0, self.r_max + self.r_bin, self.r_bin)
            self.pair_counts = np.zeros(self.r_edges.size - 1)

    def record_density(self, z):
        self.z_counts += np.histogram(z, bins=self.z_edges)[0]
        self.samples += 1

    def record_pairs(self, distances, n_pairs_ideal_per_volume):
        self.pair_counts += np.histogram(distances, bins=self.r_edges)[0]
        self._pair_norm += n_pairs_ideal_per_volume

    def density(self):
        """(z centers, n(z)) normalised so the profile integrates to N/area."""
        centers = 0.5 * (self.z_edges[1:] + self.z_edges[:-1])
        vol = self.area * self.z_bin * max(self.samples, 1)
        return centers, self.z_counts / vol

    def pair_correlation(self):
        """(r centers, g2) with ideal-gas shell normalisation."""
        centers = 0.5 * (self.r_edges[1:] + self.r_edges[:-1])
        shells = (4.0 / 3.0) * np.pi * (self.r_edges[1:] ** 3 - self.r_edges[:-1] ** 3)
        ideal = shells * self._pair_norm
        with np.errstate(invalid="ignore", divide="ignore"):
            g2 = np.where(ideal > 0, self.pair_counts / ideal, 0.0)
        return centers, g2


def make_state(positions, config):
    """Initial state: Philox stream of the seed, first noise drawn."""
    rng = np.random.Generator(np.random.Philox(config.seed))
    prev = rng.standard_normal(np.shape(positions))
    return BdState(np.array(positions, dtype=float), prev, rng)


def bd_step(state, forces, config, z_bounds=None, wrap=None):
    """One step  x += mu F dt + sqrt(kT mu dt / 2) (W_n + W_{n+1}), each
    displacement capped at max_disp; a step leaving (lo, hi) in z is redrawn
    with a fresh W_{n+1} (bd.py:101-133); periodic axes wrapped with mod."""
    drift = config.mu * config.dt * np.asarray(forces)
    amp = math.sqrt(0.5 * config.kT * config.mu * config.dt)
    shape = state.positions.shape
    for _ in range(config.max_retries + 1):
        fresh = state.rng.standard_normal(shape) if config.kT > 0 else np.zeros(shape)
        step = drift + amp * (state.prev_noise + fresh)
        if np.isfinite(config.max_disp):
            length = np.linalg.norm(step, axis=1, keepdims=True)
            too_long = length > config.max_disp
            if np.any(too_long):
                step = np.where(too_long, step * (config.max_disp / length), step)
        trial = state.positions + step
        inside = z_bounds is None or (np.all(trial[:, 2] > z_bounds[0])
                                      and np.all(trial[:, 2] < z_bounds[1]))
        if inside:
            if wrap is not None:
                for axis, box in enumerate(wrap):
                    if box is not None:
                        trial[:, axis] = np.mod(trial[:, axis], box)
            state.positions = trial
            state.prev_noise = fresh
            state.steps_done += 1
            return state
        state.rejections += 1
    raise RuntimeError("unrecoverable configuration: %d retries exhausted"
                       % config.max_retries)


def steric_pair_forces(positions, steric, boxes, tree=None, device=0):
    """Pairwise steric forces on the GPU (``se_steric_forces``), bd.py:246-270:
    periodic x and y, and z open (``boxes[2] is None``, the slab) or periodic
    (the triply periodic box of the g2 experiment)."""
    del tree                                   # the GPU builds its own cells
    if len(boxes) != 3 or boxes[0] is None or boxes[1] is None:
        raise NotImplementedError("steric forces: periodic x and y")
    lib = _lib.load()
    pos = _lib.as_f64(np.atleast_2d(positions)).reshape(-1, 3)
    out = np.zeros_like(pos)
    lz = 0.0 if boxes[2] is None else float(boxes[2])
    _lib.check(lib.se_steric_forces(int(device), _lib.dptr(pos), pos.shape[0],
                                    float(boxes[0]), float(boxes[1]), lz,
                                    float(steric.a), float(steric.U0),
                                    float(steric.r_m), int(steric.p),
                                    _lib.dptr(out)))
    return out


def wall_steric_forces(positions, steric, H):
    """Repulsion from mirror particles behind both walls, z only
    (bd.py:273-279)."""
    z = np.asarray(positions)[:, 2]
    out = np.zeros(np.shape(positions))
    out[:, 2] = steric_force(2.0 * z, steric) - steric_force(2.0 * (H - z), steric)
    return out


def bd_run(solver, steric, config, steps=None, state=None):
    """The BD loop of ``cmd_bd`` (cli.py:199-215) without its file output:
    forces = q E from the solver (need_energy=False) + steric pair forces +
    mirror-wall forces, then one :func:`bd_step` with the z margin
    n_sigma g_w and xy wrap.  Returns the state after ``steps`` steps."""
    system, params = solver.system, solver.params
    geo = system.geometry
    margin = params.n_sigma * system.g_w
    if state is None:
        state = make_state(system.positions, config)
    total = config.equil_steps + config.steps if steps is None else steps
    for _ in range(total):
        res = solver.solve(positions=state.positions, need_energy=False)
        f = res.forces \
            + steric_pair_forces(state.positions, steric, (geo.Lx, geo.Ly, None),
                                 device=getattr(solver, "device", 0)) \
            + wall_steric_forces(state.positions, steric, geo.H)
        bd_step(state, f, config, z_bounds=(margin, geo.H - margin),
                wrap=(geo.Lx, geo.Ly, None))
    return state


class DeviceBd:
    """Device-resident BD run of the slab (the cmd_bd loop, cli.py:203-215,
    at scale): positions, noise and forces stay in HBM; per step one
    ``solve_device`` (need_energy=False), the steric pair forces
    (``se_steric_forces_device``) and one ``se_bd_step_device`` (forces
    q E + steric + mirror walls, Philox noise, max_disp cap, z-bound
    rejection with margin n_sigma g_w, xy wrap).  Same dynamics as
    :func:`bd_run`, but the noise is Philox4x32-10 on the device, not numpy's
    stream, so trajectories agree with the reference statistically, not
    draw for draw."""

    def __init__(self, solver, steric, config, positions=None):
        import torch
        self._torch = torch
        self.solver, self.steric, self.config = solver, steric, config
        system, params = solver.system, solver.params
        geo = system.geometry
        self.geo = geo
        self.dev = torch.device("cuda", solver.device)
        self.stream = torch.cuda.current_stream(self.dev)
        solver.set_stream(self.stream.cuda_stream)
        self.n = n = int(system.charges.size)
        pos = system.positions if positions is None else positions
        f64 = torch.float64
        self.pos = torch.as_tensor(np.ascontiguousarray(pos, dtype=np.float64)).to(self.dev).contiguous()
        self.q = torch.as_tensor(np.ascontiguousarray(system.charges, dtype=np.float64)).to(self.dev)
        self.prev = torch.empty((n, 3), dtype=f64, device=self.dev)
        self.E = torch.empty((n, 3), dtype=f64, device=self.dev)
        self.phi = torch.empty(n, dtype=f64, device=self.dev)
        self.fst = torch.empty((n, 3), dtype=f64, device=self.dev)
        self.draws = ctypes.c_uint64(0)
        self.rejections = ctypes.c_int64(0)
        margin = params.n_sigma * system.g_w
        self.k = _lib.SeBdParams(
            dt=config.dt, mu=config.mu, kT=config.kT,
            max_disp=config.max_disp if np.isfinite(config.max_disp) else 1e300,
            z_lo=margin, z_hi=geo.H - margin, Lx=geo.Lx, Ly=geo.Ly, H=geo.H,
            a=steric.a, U0=steric.U0, r_m=steric.r_m, p=steric.p, wall=1, has_zb=1,
            max_retries=config.max_retries, seed=config.seed)
        self._lib = _lib.load()
        _lib.check(self._lib.se_bd_first_noise_device(
            self.dev.index, ctypes.c_void_p(self.stream.cuda_stream), n, config.seed,
            ctypes.c_void_p(self.prev.data_ptr())))
        self.steps_done = 0

    def step(self, steps=1):
        lib, st = self._lib, ctypes.c_void_p(self.stream.cuda_stream)
        s, g = self.steric, self.geo
        for _ in range(steps):
            self.solver.solve_device(self.pos.data_ptr(), self.phi.data_ptr(),
                                     self.E.data_ptr(), self.n, need_energy=False,
                                     graph=True)
            _lib.check(lib.se_steric_forces_device(
                self.dev.index, st, ctypes.c_void_p(self.pos.data_ptr()), self.n, g.Lx, g.Ly,
                0.0, 0.0, g.H, s.a, s.U0, s.r_m, s.p, ctypes.c_void_p(self.fst.data_ptr())))
            _lib.check(lib.se_bd_step_device(
                self.dev.index, st, ctypes.c_void_p(self.pos.data_ptr()),
                ctypes.c_void_p(self.prev.data_ptr()), ctypes.c_void_p(self.E.data_ptr()),
                ctypes.c_void_p(self.q.data_ptr()), ctypes.c_void_p(self.fst.data_ptr()),
                self.n, ctypes.byref(self.k), ctypes.byref(self.draws),
                ctypes.byref(self.rejections)))
            self.steps_done += 1
        return self

    def positions(self):
        self._torch.cuda.synchronize(self.dev)
        return self.pos.cpu().numpy()


def __getattr__(name):
    # bd.py:297 hosts the triply periodic solver in the reference
    if name == "TriplyPeriodicSolver":
        from .periodic import TriplyPeriodicSolver
        return TriplyPeriodicSolver
    raise AttributeError(name)


__all__ = ["StericParams", "BdConfig", "BdState", "Observables", "DeviceBd", "lj_force", "steric_force",
           "steric_energy", "make_state", "bd_step", "steric_pair_forces",
           "wall_steric_forces", "bd_run", "TriplyPeriodicSolver"]
