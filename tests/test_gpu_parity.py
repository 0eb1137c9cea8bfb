"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle and
the reference-generated golden fixtures.

Tolerances (north star): stencil / partition / pair membership bit-exact;
phi, E and U within 1e-10 relative L2 in fp64.  Per-stage buffers are
compared at 1e-11 (differences are summation order and erf/exp ulps only).
"""

import os

import numpy as np
import pytest

os.environ.setdefault("SE_KEEP_STAGES", "1")

from oracle import slab_oracle as O                              # noqa: E402
from paper_2101_07088_b200 import workloads as W                 # noqa: E402
from paper_2101_07088_b200.geometry import (ChargeSystem,        # noqa: E402
                                            SlabGeometry, SurfaceCharge)
from paper_2101_07088_b200.params import plan_grid               # noqa: E402
from _golden import rel_l2, solves, stages                       # noqa: E402

pytestmark = pytest.mark.gpu

TOL = 1e-10
STAGE_TOL = 1e-11
# field grids after the inverse xy FFT carry FFT rounding amplified by i k
# (|k| up to pi/h): ~3e-11 relative between cuFFT and pocketfft
FIELD_TOL = 1e-9


def _solver(system, params, refine=1):
    from paper_2101_07088_b200.slab import SlabSolver
    return SlabSolver(system, params, refine=refine)


def _compare(res, ref, forces=True, tol=TOL):
    phi, E, U, diag = ref
    assert rel_l2(res.phi_bar, phi) < tol, rel_l2(res.phi_bar, phi)
    if forces:
        assert rel_l2(res.E_bar, E) < tol, rel_l2(res.E_bar, E)
    assert abs(res.U - U) <= tol * max(1.0, abs(U)), (res.U, U)
    assert abs(res.diagnostics["B_i"] - diag["B_i"]) <= tol * max(
        1.0, abs(diag["B_i"]))


def _tiny():
    g = stages()
    geo = SlabGeometry(1.5, 1.5, 1.0, 1.0, 0.05, 0.02)
    system = ChargeSystem(geo, g["positions"], g["charges"], 0.03)
    params = plan_grid(geo, 0.03, 1e-4, Nxy=24)
    return g, system, params


def test_stages_tiny_against_oracle():
    g, system, params = _tiny()
    solver = _solver(system, params)
    res = solver.solve()
    cap = {}
    ref = O.OracleSlabSolver(system, params).solve(capture=cap)
    nx, ny, nz = params.Nx, params.Ny, params.Nz
    nyh = ny // 2 + 1
    rho = solver.debug_fetch(0).reshape(nz, 2, nx, ny).transpose(1, 2, 3, 0)
    assert rel_l2(rho[0], cap["rho_over"]) < STAGE_TOL
    assert rel_l2(rho[1], cap["rho_in"]) < STAGE_TOL
    keep = solver.debug_fetch(1).view(np.complex128).reshape(nz, 2, nx, nyh)
    psi = keep.transpose(1, 2, 3, 0)
    assert rel_l2(psi[0], cap["psi_o"][:, :nyh]) < STAGE_TOL
    assert rel_l2(psi[1], cap["psi_i"][:, :nyh]) < STAGE_TOL
    mism = solver.debug_fetch(3).view(np.complex128).reshape(4, nx, nyh)
    for i, key in enumerate(("phi_b", "e_b", "phi_t", "e_t")):
        assert rel_l2(mism[i], cap["mismatch"][key][:, :nyh]) < STAGE_TOL
    fields = solver.debug_fetch(2).reshape(nz, 4, nx, ny).transpose(1, 2, 3, 0)
    A_i = cap["k0"]["A_i"]
    z = O.cheb_nodes(nz, params.z0, params.z1)
    ref_f = cap["fields"]
    assert rel_l2(fields[0] + A_i * z, ref_f[0]) < FIELD_TOL
    assert rel_l2(-fields[1], ref_f[1]) < FIELD_TOL
    assert rel_l2(-fields[2], ref_f[2]) < FIELD_TOL
    assert rel_l2(-(fields[3] + A_i), ref_f[3]) < FIELD_TOL
    _compare(res, ref)
    # and against the reference fixture itself
    assert rel_l2(res.phi_bar, g["phi"]) < TOL
    assert rel_l2(res.E_bar, g["E"]) < TOL


def test_partition_bit_exact():
    from paper_2101_07088_b200.slab import build_partition
    g, system, params = _tiny()
    part = build_partition(system.positions, system.charges, system.geometry,
                           params)
    assert np.array_equal(part.over, g["over"])
    assert np.array_equal(part.far, g["far_idx"])
    assert np.array_equal(part.image_source, g["img_src"])
    assert np.array_equal(part.image_wall, g["img_wall"])
    assert np.array_equal(part.image_positions, g["img_pos"])
    assert np.array_equal(part.image_strengths, g["img_str"])


def test_partition_c3_bit_exact(golden_dir):
    from paper_2101_07088_b200.slab import build_partition
    gp = np.load(os.path.join(golden_dir, "partition_c3.npz"))
    system, params = W.build("c3")
    part = build_partition(system.positions, system.charges, system.geometry,
                           params)
    assert np.array_equal(part.over, gp["over"])
    assert np.array_equal(part.image_source, gp["img_src"])
    assert np.array_equal(part.image_wall, gp["img_wall"])


@pytest.mark.parametrize("case", ["c1", "c2", "c3"])
def test_workloads_against_golden(case):
    gold = solves()[case]
    system, params = W.build(case)
    res = _solver(system, params).solve()
    ref = (gold["phi"], gold["E"], float(gold["U"]), {"B_i": float(gold["B_i"])})
    _compare(res, ref)
    assert abs(res.diagnostics["k0"].A_i - gold["A_i"]) <= 1e-9 * max(
        1.0, abs(gold["A_i"]))


@pytest.mark.parametrize("case", ["c2", "c3"])
def test_workloads_against_oracle(case):
    system, params = W.build(case, N=4096 if case == "c3" else None)
    res = _solver(system, params).solve()
    _compare(res, O.oracle_solve(system, params))


# ---------------------------------------------------------------------------
# flag / geometry variants against the reference fixtures
# ---------------------------------------------------------------------------
from test_oracle_golden import VARIANTS, variant_problem       # noqa: E402


@pytest.mark.parametrize("case", sorted(VARIANTS))
def test_variants_against_golden(case):
    g = solves()[case]
    system, params, kw = variant_problem(case)
    refine = kw.pop("refine", 1)
    res = _solver(system, params, refine=refine).solve(**kw)
    forces = kw.get("need_forces", True)
    ref = (g["phi"], g["E"], float(g["U"]), {"B_i": float(g["B_i"])})
    _compare(res, ref, forces=forces)
    if not forces:
        assert np.all(res.E_bar == 0.0)


def test_positions_override_against_golden():
    g = solves()["c2n256_moved"]
    system, params = W.build("c2", N=256)
    res = _solver(system, params).solve(positions=g["positions"])
    _compare(res, (g["phi"], g["E"], float(g["U"]), {"B_i": float(g["B_i"])}))


def test_unsplit_against_golden():
    import math
    from paper_2101_07088_b200.params import EwaldParams
    g = solves()["unsplit4"]
    geo = SlabGeometry(1.0, 1.0, 0.5, 1.0, 0.2, 3.0)
    system = ChargeSystem(geo, g["positions"], g["charges"], 0.05)
    g_w, h_e = 0.05, 6.0 * 0.05
    nx = int(round(1.0 / (g_w / 2.0)))
    h = 1.0 / nx
    params = EwaldParams(xi=np.inf, g_w=g_w, g_t=g_w, delta=0.0,
                         n_g=int(math.ceil(2.0 * h_e / h)), n_sigma=6.0,
                         h_xy=h, H_E=h_e, r_nf=0.0, r_cut=0.0,
                         k_max=math.pi / h, Nx=nx, Ny=nx,
                         Nz=int(math.ceil(math.pi * (0.5 + 6 * h_e) / (2 * h))),
                         z0=-3.0 * h_e, z1=0.5 + 3.0 * h_e, h_min=6 * g_w)
    res = _solver(system, params).solve(subtract_self=True)
    _compare(res, (g["phi"], g["E"], float(g["U"]), {"B_i": float(g["B_i"])}))


def test_pair_count_matches_reference_pairs(golden_dir):
    gp = np.load(os.path.join(golden_dir, "pairs_c2n512.npz"))
    system, params = W.build("c2", N=512)
    res = _solver(system, params).solve()
    assert res.diagnostics["n_pairs"] == gp["e"].size


def test_near_field_sum_against_oracle():
    from paper_2101_07088_b200.slab import near_field_sum
    system, params = W.build("c3", N=2048)
    geo = system.geometry
    ev = np.random.default_rng(4).uniform([0, 0, 0.05], [2, 2, 0.95], (300, 3))
    nf = O.NearSources(system.positions, system.charges, geo, params)
    for kernel in ("avg", "point"):
        # the reference's keyword (slab.py:184-186), positional order too
        phi, E = near_field_sum(system.positions, system.charges, geo, params,
                                ev, kernel)
        phi2, E2 = near_field_sum(system.positions, system.charges, geo,
                                  params, eval_positions=ev, kernel=kernel)
        rphi, rE = nf.evaluate(ev, kernel)
        assert rel_l2(phi, rphi) < 1e-13
        assert rel_l2(E, rE) < 1e-13
        assert np.array_equal(phi, phi2) and np.array_equal(E, E2)
    phi = near_field_sum(system.positions, system.charges, geo, params,
                         need_field=False, subtract_unsplit_self=True)
    rphi = nf.evaluate(system.positions, "avg", need_field=False,
                       subtract_unsplit=True)
    assert rel_l2(phi, rphi) < 1e-13


def test_errors_match_reference():
    system, params = W.build("c2", N=256)
    solver = _solver(system, params)
    bad = system.positions.copy()
    bad[0, 2] = params.z1 + 0.5
    with pytest.raises(ValueError, match="outside the extended z domain"):
        solver.solve(positions=bad)
    with pytest.raises(ValueError):
        solver.solve(positions=system.positions[:10])
    # a net charge breaks the k = 0 displacement balance (dpsolver.py:208)
    sysq = ChargeSystem(system.geometry, system.positions,
                        np.ones(system.n), system.g_w)
    with pytest.raises(FloatingPointError, match="k=0 coefficient mismatch"):
        _solver(sysq, params).solve()


# ---------------------------------------------------------------------------
# size-independent properties at the north-star size (C4, N = 2^20)
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def c4():
    system, params = W.build("c4")
    solver = _solver(system, params)
    return system, params, solver, solver.solve()


def test_c4_translation_by_grid_cell(c4):
    """A shift by one grid cell in x is an exact symmetry of the discrete
    operator (stencils, near-field pairs and spectra all shift)."""
    system, params, solver, base = c4
    # the gauge pins phi(0) = 0 at the fixed origin, so compare ungauged
    ref = solver.solve(need_potential=False)
    pos = system.positions.copy()
    pos[:, 0] = (pos[:, 0] + params.h_xy) % system.geometry.Lx
    moved = solver.solve(positions=pos, need_potential=False)
    assert rel_l2(moved.phi_bar, ref.phi_bar) < 1e-11
    assert rel_l2(moved.E_bar, ref.E_bar) < 1e-11
    assert abs(moved.U - ref.U) < 1e-11 * abs(ref.U)


def test_c4_charge_sign_linearity(c4):
    system, params, solver, base = c4
    neg = ChargeSystem(system.geometry, system.positions, -system.charges,
                       system.g_w)
    res = _solver(neg, params).solve()
    assert rel_l2(res.phi_bar, -base.phi_bar) < 1e-12
    assert rel_l2(res.E_bar, -base.E_bar) < 1e-12
    assert abs(res.U - base.U) < 1e-12 * abs(base.U)


def test_c4_z_reflection(c4):
    """eps_b == eps_t and a Chebyshev grid symmetric about H/2: reflecting
    z -> H - z flips Ez.  U is symmetric only to ~1e-8: the k = 0 linear
    mode averages two displacement conditions (dpsolver.py:200-205); the CPU
    oracle shows the same 1e-8 at C3 size."""
    system, params, solver, base = c4
    pos = system.positions.copy()
    pos[:, 2] = system.geometry.H - pos[:, 2]
    res = solver.solve(positions=pos, need_potential=False)
    ref = solver.solve(need_potential=False)
    assert rel_l2(res.E_bar[:, :2], ref.E_bar[:, :2]) < 1e-9
    assert rel_l2(res.E_bar[:, 2], -ref.E_bar[:, 2]) < 1e-9
    assert abs(res.U - ref.U) < 1e-6 * abs(ref.U)
    assert abs(res.diagnostics["k0"].A_i + ref.diagnostics["k0"].A_i) < 1e-9 * abs(
        ref.diagnostics["k0"].A_i)


def test_c4_work_check(c4):
    """Energy-force consistency (reference.py:124-147): the centred
    difference of U along a displacement matches F . dX.  The displacement
    follows each charge's own force, so the signal adds coherently over the
    2^20 charges while the energy jumps of pairs and stencil nodes crossing
    the cutoffs add incoherently; h is far below g_w (truncation ~(h/g_w)^2)."""
    system, params, solver, base = c4
    d = base.forces / np.linalg.norm(base.forces, axis=1, keepdims=True)
    w2 = float(np.sum(base.forces * d))
    h = 1e-6
    up = solver.solve(positions=system.positions + 0.5 * h * d, need_forces=False).U
    dn = solver.solve(positions=system.positions - 0.5 * h * d, need_forces=False).U
    w1 = -(up - dn) / h
    assert abs(w1 - w2) / abs(w2) < 1e-3


# ---------------------------------------------------------------------------
# sharded solve: the library's phases (se_shard_spread / _fields / _charges)
# for shards first > 0, driven sequentially on one GPU (one plan per shard,
# grids summed with torch between phases 1 and 2 as the NCCL all-reduce
# does across ranks), and ShardedSlabSolver itself in a one-rank group.
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("case,world", [("c2n256", 2), ("c2n256", 3),
                                        ("c3n256_gauss_sigma", 2),
                                        ("c2n256_noforce", 2)])
def test_sharded_phases_one_gpu(case, world):
    import torch
    from paper_2101_07088_b200.sharded import CudaShardEngine, shard_range
    from paper_2101_07088_b200.slab import _flags
    from test_oracle_golden import variant_problem
    system, params, kw = variant_problem(case)
    refine = kw.pop("refine", 1)
    forces = kw.get("need_forces", True)
    flags = _flags(kw.get("need_energy", True), forces,
                   kw.get("need_potential", True),
                   kw.get("subtract_self", False),
                   kw.get("include_correction", True),
                   kw.get("force_general", False))
    n = system.charges.size
    engines = [CudaShardEngine(system, params, refine=refine, device=0)
               for _ in range(world)]
    pos = [e.positions(system.positions) for e in engines]
    ranges = [shard_range(n, r, world) for r in range(world)]
    rhos = [e.spread(p, f, c, flags)
            for e, p, (f, c) in zip(engines, pos, ranges)]
    total = torch.stack(rhos).sum(0)
    for r in rhos:
        r.copy_(total)
    for e in engines:
        e.fields()
    outs = [e.charges(p, c, forces)
            for e, p, (_, c) in zip(engines, pos, ranges)]
    phi = torch.cat([o[0] for o in outs]).cpu().numpy()
    E = torch.cat([o[1] for o in outs]).cpu().numpy()
    U = sum(o[2] for o in outs)
    g = solves()[case]
    assert rel_l2(phi, g["phi"]) < TOL
    if forces:
        assert rel_l2(E, g["E"]) < TOL
    assert abs(U - g["U"]) <= TOL * max(1.0, abs(g["U"]))
    for e in engines:
        e.close()


@pytest.mark.parametrize("decompose,near", [(False, "index"), (True, "index"),
                                            (True, "cell")])
def test_sharded_solver_one_rank(decompose, near):
    import socket
    import torch.distributed as dist
    from paper_2101_07088_b200.sharded import ShardedSlabSolver
    from test_oracle_golden import variant_problem
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port,
                            rank=0, world_size=1)
    try:
        system, params, kw = variant_problem("c2n256")
        solver = ShardedSlabSolver(system, params, device=0, decompose=decompose,
                                   near=near)
        res = solver.solve(**kw)
        g = solves()["c2n256"]
        assert rel_l2(res.phi_bar, g["phi"]) < TOL
        assert rel_l2(res.E_bar, g["E"]) < TOL
        assert abs(res.U - g["U"]) <= TOL * max(1.0, abs(g["U"]))
        solver.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ranks", [2, 4])
def test_cell_routed_near_field_one_gpu(ranks):
    """The cell-routed near field of P virtual ranks on one GPU: each rank's
    sources are the charges routed to it (its x slab + r_cut halo), its
    targets those it owns; the assembled near sums, with the index-sharded
    grid pipeline of one plan, reproduce the reference solve (C3, jumps at
    both walls) and the single-GPU pair count."""
    import torch
    from paper_2101_07088_b200 import _lib
    from paper_2101_07088_b200.sharded import CudaShardEngine, cell_destinations
    from paper_2101_07088_b200.slab import _flags
    g = solves()["c3"]
    system, params = W.build("c3")
    n = system.n
    ref_pairs = _solver(system, params).solve().diagnostics["n_pairs"]
    eng = CudaShardEngine(system, params, device=0)
    dev = eng.device
    pos = torch.as_tensor(system.positions, device=dev)
    q = torch.as_tensor(system.charges, device=dev)
    flags = _flags(True, True, True, False, True, False)
    eng.spread_own(pos, 0, n, flags)
    ci, dest, tgt = cell_destinations(pos[:, 0], system.geometry.Lx, ranks,
                                      float(params.r_cut))
    geo = system.geometry
    zmin = torch.stack([pos[:, 2].min(), -pos[:, 2].max(),
                        2 * geo.H - pos[:, 2].max()]).min().reshape(1)
    near = torch.zeros((4, n), dtype=torch.float64, device=dev)
    near0 = torch.zeros(1, dtype=torch.float64, device=dev)
    pairs = 0
    for r in range(ranks):
        mine = dest == r
        idx = torch.cat([ci[mine & tgt], ci[mine & ~tgt]])
        nt = int((mine & tgt).sum())
        out, n0, npairs = eng.near(pos[idx].contiguous(), q[idx].contiguous(), nt,
                                   r == 0, zmin)
        near[:, idx[:nt]] = out
        near0 += n0
        pairs += int(npairs.item())
    eng.fields()
    phi, E, U, diag = eng.charges_own(pos, near, near0, True)
    assert pairs == ref_pairs
    assert rel_l2(phi.cpu().numpy(), g["phi"]) < TOL
    assert rel_l2(E.cpu().numpy(), g["E"]) < TOL
    assert abs(U - float(g["U"])) <= TOL * max(1.0, abs(float(g["U"])))
    eng.close()


def test_shard_phase_order():
    import ctypes
    from paper_2101_07088_b200 import _lib
    system, params = W.build("c2", N=64)
    solver = _solver(system, params)
    with pytest.raises(RuntimeError):
        _lib.check(solver._lib.se_shard_fields(solver._plan))
    with pytest.raises(RuntimeError):
        _lib.check(solver._lib.se_shard_charges(solver._plan, None, None,
                                                None, None, None))
    with pytest.raises(ValueError):
        ptr, size = ctypes.c_void_p(), ctypes.c_int64()
        _lib.check(solver._lib.se_shard_spread(
            solver._plan, None, 64, 40, 30, 0, ctypes.byref(ptr),
            ctypes.byref(size)))
    res = solver.solve()                  # a full solve still works after
    assert np.all(np.isfinite(res.phi_bar))


# ---------------------------------------------------------------------------
# fp32 mode (SE_FP32): near-field pair kernels in single precision; the pair
# set is still the exact fp64 one, results within the Ewald tolerance delta
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("case", ["c2n256", "c3n256_gauss_sigma"])
def test_fp32_mode_within_tolerance(case):
    from paper_2101_07088_b200.slab import SlabSolver
    from test_oracle_golden import variant_problem
    system, params, kw = variant_problem(case)
    kw.pop("refine", None)
    g = solves()[case]
    res = SlabSolver(system, params, precision="fp32").solve(**kw)
    delta = params.delta
    assert rel_l2(res.phi_bar, g["phi"]) < delta
    assert rel_l2(res.E_bar, g["E"]) < delta
    assert abs(res.U - g["U"]) <= delta * abs(g["U"])
    ref64 = SlabSolver(system, params).solve(**kw)
    assert res.diagnostics["n_pairs"] == ref64.diagnostics["n_pairs"]


def test_fp32_mode_rejects_unknown_precision():
    from paper_2101_07088_b200.slab import SlabSolver
    system, params = W.build("c2", N=64)
    with pytest.raises(ValueError):
        SlabSolver(system, params, precision="bf16")


# ---------------------------------------------------------------------------
# distributed grid pipeline (se_dist_*): P ranks emulated sequentially on one
# GPU, the collectives (reduce-scatter, two all-to-alls, all-reduce,
# all-gather) done with torch between the library phases
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("case,world", [("c2n256", 2), ("c2n256", 3),
                                        ("c3n256_gauss_sigma", 4),
                                        ("c2n256_noforce", 2),
                                        ("c2n256_nocorr", 3)])
def test_distributed_grid_pipeline_one_gpu(case, world):
    import torch
    from paper_2101_07088_b200.sharded import CudaShardEngine, shard_range
    from paper_2101_07088_b200.slab import _flags
    from test_oracle_golden import variant_problem
    system, params, kw = variant_problem(case)
    refine = kw.pop("refine", 1)
    forces = kw.get("need_forces", True)
    flags = _flags(kw.get("need_energy", True), forces,
                   kw.get("need_potential", True),
                   kw.get("subtract_self", False),
                   kw.get("include_correction", True),
                   kw.get("force_general", False))
    n = system.charges.size
    eng = [CudaShardEngine(system, params, refine=refine, device=0)
           for _ in range(world)]
    buf = [e.dist_setup(r, world) for r, e in enumerate(eng)]
    pos = [e.positions(system.positions) for e in eng]
    ranges = [shard_range(n, r, world) for r in range(world)]
    for e, p_, (f, c) in zip(eng, pos, ranges):
        e.spread(p_, f, c, flags)
    total = torch.stack([b["rho"] for b in buf]).sum(0)
    for r, b in enumerate(buf):                              # reduce-scatter
        k = b["rho_slab"].numel()
        b["rho_slab"].copy_(total[r * k:(r + 1) * k])

    def all_to_all(send, recv):
        for r in range(world):
            for s in range(world):
                k = buf[r][recv].numel() // world
                buf[r][recv][s * k:(s + 1) * k].copy_(buf[s][send][r * k:(r + 1) * k])
    for e in eng:
        e.dist_forward()
    all_to_all("send_fwd", "recv_fwd")
    for e in eng:
        e.dist_modes()
    all_to_all("send_back", "recv_back")
    dsc = torch.stack([b["dsc"] for b in buf]).sum(0)        # all-reduce
    for b in buf:
        b["dsc"].copy_(dsc)
    for e in eng:
        e.dist_fields()
    slabs = torch.cat([b["fields_slab"] for b in buf])       # all-gather
    for b in buf:
        b["fields"].copy_(slabs)
    outs = [e.charges(p_, c, forces) for e, p_, (_, c) in zip(eng, pos, ranges)]
    phi = torch.cat([o[0] for o in outs]).cpu().numpy()
    E = torch.cat([o[1] for o in outs]).cpu().numpy()
    U = sum(o[2] for o in outs)
    g = solves()[case]
    assert rel_l2(phi, g["phi"]) < TOL
    if forces:
        assert rel_l2(E, g["E"]) < TOL
    assert abs(U - g["U"]) <= TOL * max(1.0, abs(g["U"]))
    for e in eng:
        e.close()


@pytest.mark.gpu
def test_freespace_slab_agreement():
    """The reference's `validate --suite freespace` (validate.py:110-132,
    PAPER Table 2): L = 28 and 32 solves extrapolated to L = infinity against
    the 400-image open-slab field; the GPU fields match the reference's
    solver to 1e-10 and the extrapolated error is its 9.755e-6 (<= 5e-5)."""
    import warnings
    from paper_2101_07088_b200 import ChargeSystem, SlabGeometry, plan_grid
    from paper_2101_07088_b200.slab import SlabSolver
    G = np.load(os.path.join(os.path.dirname(__file__), "golden", "freespace.npz"))
    fields = {}
    for L in (28.0, 32.0):
        geo = SlabGeometry(L, L, 2.0, eps=1.0, eps_b=0.5, eps_t=0.2)
        pos = G["charges"].copy()
        pos[:, :2] += 0.5 * L
        system = ChargeSystem(geo, pos, G["q"], 1e-2)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            params = plan_grid(geo, 1e-2, 1e-4, xi=3.0177, h_min=0.01, strict=False)
        fields[L] = SlabSolver(system, params).solve().E_bar
        ref = G["E_L%d" % int(L)]
        assert np.linalg.norm(fields[L] - ref) <= 1e-10 * np.linalg.norm(ref)
    e_inf = (32.0 * fields[32.0] - 28.0 * fields[28.0]) / 4.0   # reference.py:78-80
    e_f = G["e_f"]
    err = np.max(np.abs(e_inf - e_f)) / np.mean(np.linalg.norm(e_f, axis=1))
    assert err <= 5e-5
    assert abs(err - float(G["err"])) <= 1e-3 * float(G["err"])


@pytest.mark.gpu
@pytest.mark.parametrize("fused", ["0", "1", "0-overflow"])
def test_both_near_field_paths_against_goldens(fused):
    """The near field has two kernels chosen by size (fused one-warp-per-
    point below 40000 points, scan -> lists -> eval above): force each on
    the golden workloads and the exact pair count (SE_NEAR_FUSED is read
    once per process, hence the subprocess)."""
    import subprocess
    import sys
    env = dict(os.environ, SE_NEAR_FUSED=fused[0])
    if fused.endswith("overflow"):
        # lists far too short: most points overflow and are evaluated by the
        # device-side fallback (fused kernel over the overflow list)
        env["SE_NEAR_LIST_SCALE"] = "0.05"
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-x",
                        os.path.join(here, "test_gpu_parity.py"), "-k",
                        "workloads_against_golden or pair_count or near_field_sum "
                        "or variants_against_golden"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.gpu
@pytest.mark.parametrize("layout", ["xy3", "xy4_z8", "tmap0"])
def test_alternative_layouts_against_goldens(layout):
    """The measured-and-kept-off layout switches stay correct: near-field
    columns of r_c / 3 or r_c / 4 (7 x 7 / 9 x 9 column walks), z bins of
    r_c / 8, and the contiguous DCT warp-tile map, on the list path, against
    the goldens and the exact pair count (env switches are read once per
    process, hence the subprocess)."""
    import subprocess
    import sys
    extra = {"xy3": {"SE_CELL_XYDIV": "3"},
             "xy4_z8": {"SE_CELL_XYDIV": "4", "SE_CELL_ZDIV": "8"},
             "tmap0": {"SE_DCT_TMAP": "0"}}[layout]
    env = dict(os.environ, SE_NEAR_FUSED="0", **extra)
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-x",
                        os.path.join(here, "test_gpu_parity.py"), "-k",
                        "workloads_against_golden or pair_count or variants_against_golden"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_graph_replay_matches_direct_solve():
    """SE_GRAPH: the warm solve, the capture and the replays give the same
    results as direct solves, also after the positions change in place."""
    import torch
    system, params = W.build("c3", N=4096)
    n = system.n
    s = _solver(system, params)
    s.set_stream(torch.cuda.current_stream().cuda_stream)
    pos = torch.as_tensor(system.positions, device="cuda").contiguous()
    phi = torch.empty(n, dtype=torch.float64, device="cuda")
    E = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    direct = s.solve()
    for _ in range(4):                       # warm, capture, replay, replay
        U, diag = s.solve_device(pos.data_ptr(), phi.data_ptr(), E.data_ptr(), n, graph=True)
        torch.cuda.synchronize()
        assert np.array_equal(phi.cpu().numpy(), direct.phi_bar)
        assert np.array_equal(E.cpu().numpy(), direct.E_bar)
        assert U == direct.U
    moved = system.positions.copy()
    moved[:, :2] = (moved[:, :2] + 0.013) % 2.0
    pos.copy_(torch.as_tensor(moved))
    U, diag = s.solve_device(pos.data_ptr(), phi.data_ptr(), E.data_ptr(), n, graph=True)
    torch.cuda.synchronize()
    ref = s.solve(positions=moved)
    assert np.array_equal(phi.cpu().numpy(), ref.phi_bar)
    assert U == ref.U


# ---------------------------------------------------------------------------
# repeated host-API solves replay the captured CUDA graph (SlabSolver.solve
# graph=True, the default): every flag / geometry variant -- surface charge
# (wall energy), no jump, no correction, potential or forces only, self
# subtraction -- gives the reference's result on the replays too, and a
# replay on moved positions gives the moved-positions golden
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("case", ["c2n256", "c2n256_noforce", "c2n256_nopot",
                                  "c2n256_selfsub", "c2n256_nocorr", "c2n256_nojump",
                                  "c2n256_general", "c2n256_nojump_sigma",
                                  "c3n256_gauss_sigma", "c3n512_vacuum_metal"])
def test_graph_replay_variants(case):
    from test_oracle_golden import variant_problem
    gold = solves()
    system, params, kw = variant_problem(case)
    refine = kw.pop("refine", 1)
    solver = _solver(system, params, refine=refine)
    g = gold[case]
    ref = (g["phi"], g["E"], float(g["U"]), {"B_i": float(g["B_i"])})
    outs = [solver.solve(**kw) for _ in range(4)]      # warm, capture, 2 replays
    for res in outs:
        _compare(res, ref, forces=kw.get("need_forces", True))
    assert outs[2].U == outs[3].U
    solver.close()


def test_graph_replay_moved_positions():
    gold = solves()
    g = gold["c2n256_moved"]
    system, params = W.build("c2", N=256)
    solver = _solver(system, params)
    for _ in range(3):                                 # warm, capture, replay
        solver.solve()
    res = solver.solve(positions=g["positions"])       # replay, new positions
    _compare(res, (g["phi"], g["E"], float(g["U"]), {"B_i": float(g["B_i"])}))
    solver.close()
