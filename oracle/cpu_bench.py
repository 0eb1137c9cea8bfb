"""TEST INFRASTRUCTURE — bounded CPU timing of the oracle for ``bench.py``.

The full reference-style solve at the north-star size (N = 2^20 charges on
a 256 x 256 x 258 grid) takes ~20 minutes on one core and does not fit in
memory (the near field alone materialises ~6e8 pairs).
``bench.py``'s CPU-baseline leg therefore times the oracle stage by stage on a
bounded sample of the same workload and extrapolates linearly in the charge
count (the per-charge stages are independent per charge):

* grid stages (xy FFT + DCT-I, mode BVPs with refinement, correction,
  inverse transforms) on the FULL grid once;
* spreading of a sample of sources (charges + images) — per source cost;
* interpolation of the 4 fields at a sample of charges — per charge cost;
* near field of a sample of target charges against ALL sources (full
  density, the KD-tree over all 3N sources is built) — per target cost.

The result is seconds per full solve = grid + N_src * t_spread + N * (t_interp
+ t_near).  ``workers`` mirrors the reference's ``SlabSolver(threads=T)``
(sw/slab.py:197, scipy.fft workers of the xy transforms, slab.py:242,250);
every other stage is single-threaded numpy in the reference too.
"""

import time

import numpy as np

from . import slab_oracle as O


def _time(fn, *a, **kw):
    t = time.perf_counter()
    out = fn(*a, **kw)
    return time.perf_counter() - t, out


def grid_stage_seconds(system, params, workers=1):
    """Wall time of the oracle's grid pipeline on the full grid (jump path)."""
    solver = O.OracleSlabSolver(system, params, workers=workers)
    geo, par = system.geometry, params
    rng = np.random.default_rng(1)
    shape = solver.grid.shape
    rho_o = rng.standard_normal(shape)
    rho_i = rng.standard_normal(shape)
    t0 = time.perf_counter()
    both = solver.modes.solve(np.stack([solver._forward(rho_o),
                                        solver._forward(rho_i)]))
    psi_o, psi_i = both[0], both[1]
    dpsi_i = O.cheb_deriv(psi_i, par.z0, par.z1)
    dpsi_o = O.cheb_deriv(psi_o, par.z0, par.z1)
    T0, TH = solver.t_wall[0.0], solver.t_wall[geo.H]
    cb, ct = geo.exterior_factor_bottom(), geo.exterior_factor_top()
    mism = {"phi_b": psi_i @ T0 - cb * (psi_o @ T0),
            "e_b": geo.eps * (dpsi_i @ T0) - geo.eps_b * cb * (dpsi_o @ T0),
            "phi_t": psi_i @ TH - ct * (psi_o @ TH),
            "e_t": geo.eps * (dpsi_i @ TH) - geo.eps_t * ct * (dpsi_o @ TH)}
    corr, dcorr = solver._apply_correction(mism)
    vals = O.cheb_values(psi_i) + corr
    solver._to_grid(vals)
    dz = O.cheb_values(dpsi_i) + dcorr
    solver._to_grid(vals * solver.ikx[:, None, None])
    solver._to_grid(vals * solver.iky[None, :, None])
    solver._to_grid(dz)
    return time.perf_counter() - t0


def per_charge_seconds(system, params, sample=4096, seed=3):
    """(t_spread per source, t_interp per charge, t_near per target) from a
    sample of the workload's own charges."""
    solver = O.OracleSlabSolver(system, params)
    par, geo = params, system.geometry
    pos, q = system.positions, system.charges
    rng = np.random.default_rng(seed)
    pick = rng.choice(pos.shape[0], size=min(sample, pos.shape[0]),
                      replace=False)
    t_sp, _ = _time(solver.grid.spread, pos[pick], q[pick], par.g_t, par.H_E,
                    par.H_E)
    fields = np.zeros((4,) + solver.grid.shape)
    t_in, _ = _time(solver.grid.interpolate, fields, pos[pick], par.g_t,
                    par.H_E, par.H_E)
    nf = O.NearSources(pos, q, geo, par)               # full-density sources
    t_nf, _ = _time(nf.evaluate, pos[pick[:max(1, len(pick) // 4)]], "avg")
    n_s = len(pick)
    return t_sp / n_s, t_in / n_s, t_nf / max(1, len(pick) // 4)


def estimate_solve_seconds(system, params, sample=4096, grid_seconds=None,
                           workers=1):
    """Extrapolated seconds of one full oracle solve and the stage parts."""
    if grid_seconds is None:
        grid_seconds = grid_stage_seconds(system, params, workers=workers)
    t_sp, t_in, t_nf = per_charge_seconds(system, params, sample)
    n = system.n
    z = system.positions[:, 2]
    n_img = int(np.count_nonzero((z < 2 * params.H_E)
                                 | (z > system.geometry.H - 2 * params.H_E)))
    n_src = n + n_img
    total = grid_seconds + n_src * t_sp + n * (t_in + t_nf)
    return {"total_s": total, "grid_s": grid_seconds,
            "spread_s_per_source": t_sp, "interp_s_per_charge": t_in,
            "near_s_per_charge": t_nf, "n_sources": n_src,
            "sample_charges": int(min(sample, n))}
