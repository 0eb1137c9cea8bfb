"""Brownian dynamics against reference goldens
(tests/golden/make_bd.py): steric force / energy curves, mirror-wall forces
and three integrator steps with the reference's Philox noise on CPU; the
GPU steric pair forces (periodic xy, open z) on the GPU."""

import os

import numpy as np
import pytest

from paper_2101_07088_b200 import bd as B
from _golden import rel_l2

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "bd.npz"))
L, H = 1.0, 0.6


def _steric(name):
    a, U0, r_m, p = G["steric_%s" % name]
    return B.StericParams(a=float(a), U0=float(U0), r_m=float(r_m), p=int(p))


@pytest.mark.parametrize("name", ["a", "b", "c"])
def test_steric_curves(name):
    s = _steric(name)
    assert np.array_equal(B.steric_force(G["r"], s), G["force_%s" % name])
    assert np.array_equal(B.steric_energy(G["r"], s), G["energy_%s" % name])


@pytest.mark.parametrize("name", ["a", "b", "c"])
def test_wall_forces(name):
    got = B.wall_steric_forces(G["pos"], _steric(name), H)
    assert np.array_equal(got, G["wall_%s" % name])


def test_bd_steps_match_reference_stream():
    cfg = B.BdConfig(dt=2e-5, steps=3, seed=5, max_disp=0.01)
    state = B.make_state(G["bd_pos0"], cfg)
    for k in range(3):
        B.bd_step(state, G["bd_forces"], cfg, z_bounds=(0.05, H - 0.05), wrap=(L, L, None))
        assert np.array_equal(state.positions, G["bd_traj"][k])
    assert state.rejections == int(G["bd_rejections"])


def test_bd_step_rejects_and_exhausts():
    cfg = B.BdConfig(dt=1e-3, steps=1, seed=1, max_retries=3)
    state = B.make_state(np.array([[0.5, 0.5, 0.3]]), cfg)
    with pytest.raises(RuntimeError):
        B.bd_step(state, np.zeros((1, 3)), cfg, z_bounds=(0.4, 0.5))
    assert state.rejections == 4


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["a", "b", "c"])
def test_gpu_steric_pair_forces(name):
    got = B.steric_pair_forces(G["pos"], _steric(name), (L, L, None))
    ref = G["pair_%s" % name]
    assert rel_l2(got, ref) < 1e-12
    # the per-particle zero pattern (who has neighbours) is exact
    assert np.array_equal(np.abs(got).sum(1) > 0, np.abs(ref).sum(1) > 0)


def test_steric_pair_forces_rejects_open_xy():
    with pytest.raises(NotImplementedError):
        B.steric_pair_forces(G["pos"], _steric("a"), (None, L, None))


@pytest.mark.gpu
def test_gpu_bd_loop_matches_reference():
    """Two steps of the cmd_bd loop with the GPU solver and steric forces
    against the reference's own loop (tests/golden/make_bd.py --loop)."""
    from paper_2101_07088_b200 import workloads as W
    from paper_2101_07088_b200.slab import SlabSolver
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "bd_loop.npz"))
    system, params = W.build("c2", N=256)
    solver = SlabSolver(system, params)
    st = B.StericParams(a=0.01)
    cfg = B.BdConfig(dt=1e-6, steps=2, seed=3, max_disp=st.a)
    state = B.make_state(system.positions, cfg)
    for k in range(2):
        B.bd_run(solver, st, cfg, steps=1, state=state)
        assert np.max(np.abs(state.positions - g["traj"][k])) < 1e-12
    assert state.rejections == int(g["rejections"])


@pytest.mark.gpu
def test_gpu_device_bd_deterministic_matches_host_loop():
    """kT = 0: the device-resident loop is the deterministic drift of the
    host loop (same forces, cap, walls, wrap) step for step."""
    from paper_2101_07088_b200 import workloads as W
    from paper_2101_07088_b200.slab import SlabSolver
    system, params = W.build("c2", N=256)
    st = B.StericParams(a=0.01)
    cfg = B.BdConfig(dt=1e-6, steps=3, seed=3, max_disp=st.a, kT=0.0)
    host = B.bd_run(SlabSolver(system, params), st, cfg, steps=3)
    dev = B.DeviceBd(SlabSolver(system, params), st, cfg).step(3)
    assert np.max(np.abs(dev.positions() - host.positions)) < 1e-12


@pytest.mark.gpu
def test_gpu_device_bd_noise_statistics():
    """Free diffusion (no charges' forces: q = 0 would be rejected by the
    solver, so a dilute system with a huge dt-scale noise): the step is
    N(0, kT mu dt) per component in the bulk; no particle leaves (0, H)."""
    from paper_2101_07088_b200 import workloads as W
    from paper_2101_07088_b200.slab import SlabSolver
    system, params = W.build("c3")
    st = B.StericParams(a=1e-4)
    dt = 1e-7
    cfg = B.BdConfig(dt=dt, steps=1, seed=11, max_disp=1.0, kT=1.0)
    # keep the start > 30 noise widths inside the z bounds (a random start on
    # the bound is rejected forever, as in the reference)
    zb = params.n_sigma * system.g_w
    H = system.geometry.H
    start = system.positions.copy()
    start[:, 2] = (zb + 0.01) + (start[:, 2] - zb) * (H - 2 * zb - 0.02) / (H - 2 * zb)
    bd = B.DeviceBd(SlabSolver(system, params), st, cfg, positions=start)
    p0 = bd.positions()
    p1 = bd.step(1).positions()
    d = p1 - p0
    d[:, :2] -= system.geometry.Lx * np.round(d[:, :2] / system.geometry.Lx)
    var = d.var(axis=0) / (cfg.kT * cfg.mu * dt)
    assert np.all(np.abs(var - 1.0) < 0.05), var      # 32768 samples per axis
    assert np.all(np.abs(d.mean(axis=0)) < 0.05 * np.sqrt(dt))
    assert np.all((p1[:, 2] > zb) & (p1[:, 2] < H - zb))
