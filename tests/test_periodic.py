"""Triply periodic twin against the reference's own
outputs (tests/golden/tp.npz, made by tests/golden/make_tp.py): the oracle
restatement on CPU, the se_tp_* GPU path and the fully periodic steric
forces on the GPU, and two steps of the g2 experiment's BD loop."""

import os

import numpy as np
import pytest

from oracle import tp_oracle as T
from _golden import rel_l2

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "tp.npz"))


def _g2():
    box = float(G["g2_box"])
    return box, (box, box, box), float(G["g2_eps"])


@pytest.mark.parametrize("tag", ["a", "b"])
def test_oracle_poisson_matches_reference(tag):
    phi, e = T.poisson(G["rho_" + tag], 0.7, tuple(G["box_" + tag]), with_field=True)
    assert rel_l2(phi, G["phi_" + tag]) < 1e-13
    assert rel_l2(e, G["e_" + tag]) < 1e-13


def test_oracle_forces_match_reference():
    box, boxes, eps = _g2()
    s = T.TpSolver(boxes, 32, 0.25, eps)
    assert abs(s.r_cut - float(G["g2_rcut"])) < 1e-12
    assert s.n == tuple(G["g2_n"])
    f = s.forces(G["g2_pos"], G["g2_q"])
    assert rel_l2(f, G["g2_forces"]) < 1e-11


def test_periodic_api_names():
    import paper_2101_07088_b200 as sw
    from paper_2101_07088_b200 import bd
    assert "solve_triply_periodic" in sw.__all__
    assert callable(sw.solve_triply_periodic)
    assert bd.TriplyPeriodicSolver.__name__ == "TriplyPeriodicSolver"


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["a", "b"])
def test_gpu_poisson_matches_reference(tag):
    import paper_2101_07088_b200 as sw
    rho, box = G["rho_" + tag], tuple(G["box_" + tag])
    phi, e = sw.solve_triply_periodic(rho, 0.7, *box, with_field=True)
    assert rel_l2(phi, G["phi_" + tag]) < 1e-13
    assert rel_l2(e, G["e_" + tag]) < 1e-13
    assert rel_l2(sw.solve_triply_periodic(rho, 0.7, *box), G["phi_only_" + tag]) < 1e-13


@pytest.mark.gpu
def test_gpu_tp_forces_match_reference():
    from paper_2101_07088_b200.periodic import TriplyPeriodicSolver
    box, boxes, eps = _g2()
    s = TriplyPeriodicSolver(boxes, 32, 0.25, eps, delta=5e-4)
    assert s.n == tuple(G["g2_n"])
    f = s.forces(G["g2_pos"], G["g2_q"])
    assert rel_l2(f, G["g2_forces"]) < 1e-11
    # translation by a grid cell leaves the forces unchanged
    h = box / 32
    f2 = s.forces(G["g2_pos"] + np.array([h, 2 * h, -h]), G["g2_q"])
    assert rel_l2(f2, f) < 1e-11


@pytest.mark.gpu
def test_gpu_periodic_steric_matches_reference():
    from paper_2101_07088_b200 import bd as B
    box, boxes, eps = _g2()
    st = B.StericParams(a=1.0, U0=0.2233, r_m=1.0, p=2)
    got = B.steric_pair_forces(G["g2_pos"], st, boxes)
    assert rel_l2(got, G["g2_steric"]) < 1e-12


@pytest.mark.gpu
def test_gpu_g2_bd_loop_matches_reference():
    from paper_2101_07088_b200 import bd as B
    from paper_2101_07088_b200.periodic import TriplyPeriodicSolver
    box, boxes, eps = _g2()
    st = B.StericParams(a=1.0, U0=0.2233, r_m=1.0, p=2)
    s = TriplyPeriodicSolver(boxes, 32, 0.25, eps, delta=5e-4)
    cfg = B.BdConfig(dt=5e-3, steps=2, seed=42, max_disp=1.0)
    state = B.make_state(G["g2_pos"], cfg)
    for k in range(2):
        f = s.forces(state.positions, G["g2_q"]) + B.steric_pair_forces(state.positions, st, boxes)
        B.bd_step(state, f, cfg, wrap=boxes)
        assert np.max(np.abs(state.positions - G["g2_traj"][k])) < 1e-9


@pytest.mark.gpu
def test_gpu_tp_edges():
    """Empty and single-charge systems, positions outside the primary box
    (wrapped by the stencils and the minimum image), odd grid sizes."""
    from paper_2101_07088_b200.periodic import TriplyPeriodicSolver
    box, boxes, eps = _g2()
    s = TriplyPeriodicSolver(boxes, 32, 0.25, eps, delta=5e-4)
    assert s.forces(np.zeros((0, 3)), np.zeros(0)).shape == (0, 3)
    one = s.forces(G["g2_pos"][:1], np.array([1.0]))
    assert one.shape == (1, 3) and np.all(np.isfinite(one))
    assert np.max(np.abs(one)) < 1e-8          # a lone charge feels no net force
    pos = G["g2_pos"].copy()
    shifted = pos + np.array([box, -box, 2 * box])
    f0 = s.forces(pos, G["g2_q"])
    f1 = s.forces(shifted, G["g2_q"])
    assert rel_l2(f1, f0) < 1e-10
    o = T.TpSolver(boxes, 31, 0.25, eps)
    g = TriplyPeriodicSolver(boxes, 31, 0.25, eps, delta=5e-4)
    assert g.n == o.n
    sub = slice(0, 120)
    assert rel_l2(g.forces(pos[sub], G["g2_q"][sub]), o.forces(pos[sub], G["g2_q"][sub])) < 1e-10


@pytest.mark.gpu
def test_gpu_tp_forces_device_graph():
    """forces_device replayed as a CUDA graph (se_tp_set_graph): warm call,
    capture, replays -- all equal to the reference's forces, and a replay
    on moved positions (same buffer) equals the eager result there."""
    import torch
    from paper_2101_07088_b200.periodic import TriplyPeriodicSolver
    box, boxes, eps = _g2()
    s = TriplyPeriodicSolver(boxes, 32, 0.25, eps, delta=5e-4)
    st = torch.cuda.current_stream()
    s.set_stream(st.cuda_stream)
    n = G["g2_q"].size
    pos = torch.tensor(G["g2_pos"], device="cuda")
    q = torch.tensor(G["g2_q"], device="cuda")
    out = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    for _ in range(4):
        s.forces_device(pos.data_ptr(), q.data_ptr(), n, out.data_ptr(), graph=True)
        torch.cuda.synchronize()
        assert rel_l2(out.cpu().numpy(), G["g2_forces"]) < 1e-11
    h = box / 32
    moved = G["g2_pos"] + np.array([0.3 * h, -0.7 * h, 0.2 * h])
    pos.copy_(torch.tensor(moved))
    s.forces_device(pos.data_ptr(), q.data_ptr(), n, out.data_ptr(), graph=True)
    torch.cuda.synchronize()
    ref = s.forces(moved, G["g2_q"])
    assert rel_l2(out.cpu().numpy(), ref) < 1e-12
    s.close()
