"""Sharded solve (charges split by index across ranks, grids all-reduced):
the host logic of ``ShardedSlabSolver`` on CPU over ``gloo`` with
world_size 2 and 3, each rank's phases computed by the oracle engine.  The
result must equal the unsharded solve (and the reference's golden output)
up to the summation order of the grids.  The GPU engine is covered by
``test_gpu_parity.py::test_sharded_solver_one_rank``."""

import os
import pickle
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from _golden import rel_l2, solves
from paper_2101_07088_b200.sharded import ShardedSlabSolver, shard_range

CASES = ["c2n256", "c2n256_noforce", "c2n256_nocorr", "c3n256_gauss_sigma"]
TOL = 1e-12


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cases, outdir, near="index"):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    for p in (here, os.path.dirname(here)):
        if p not in sys.path:
            sys.path.insert(0, p)
    from _oracle_engine import OracleShardEngine
    from test_oracle_golden import variant_problem
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port,
                            rank=rank, world_size=world)
    try:
        out = {}
        for case in cases:
            system, params, kw = variant_problem(case)
            refine = kw.pop("refine", 1)
            eng = OracleShardEngine(system, params, refine=refine)
            solver = ShardedSlabSolver(system, params, engine=eng, near=near)
            res = solver.solve(**kw)
            out[case] = (res.phi_bar, res.E_bar, res.U,
                         res.diagnostics["B_i"], solver.first, solver.count)
        with open(os.path.join(outdir, "rank%d.pkl" % rank), "wb") as f:
            pickle.dump(out, f)
    finally:
        dist.destroy_process_group()


def test_shard_ranges_cover():
    for n in (0, 1, 5, 256, 1 << 20):
        for w in (1, 2, 3, 8):
            got = [shard_range(n, r, w) for r in range(w)]
            assert got[0][0] == 0
            for (f0, c0), (f1, _) in zip(got, got[1:]):
                assert f0 + c0 == f1
            assert got[-1][0] + got[-1][1] == n
            assert max(c for _, c in got) - min(c for _, c in got) <= 1


@pytest.mark.parametrize("world,cases,near", [(2, CASES, "index"),
                                              (3, ["c3n256_gauss_sigma"], "index"),
                                              (2, ["c2n256", "c2n256_noforce"], "cell"),
                                              (3, ["c2n256_nocorr"], "cell")])
def test_sharded_matches_golden(tmp_path, world, cases, near):
    """Index-sharded spread; near field either with every charge as a source
    on every rank (index) or routed by x slab with an r_cut halo (cell)."""
    mp.spawn(_worker, args=(world, _free_port(), cases, str(tmp_path), near),
             nprocs=world, join=True)
    gold = solves()
    ranks = []
    for r in range(world):
        with open(tmp_path / ("rank%d.pkl" % r), "rb") as f:
            ranks.append(pickle.load(f))
    for case in cases:
        g = gold[case]
        phi0, E0, U0, B0, _, _ = ranks[0][case]
        assert rel_l2(phi0, g["phi"]) < TOL, case
        if "noforce" not in case:
            assert rel_l2(E0, g["E"]) < TOL, case
        assert abs(U0 - g["U"]) <= TOL * max(1.0, abs(g["U"])), case
        assert abs(B0 - g["B_i"]) <= TOL * max(1.0, abs(g["B_i"])), case
        # every rank returns the same gathered result and the same energy
        for r in range(1, world):
            phi, E, U, B, first, count = ranks[r][case]
            assert np.array_equal(phi, phi0) and np.array_equal(E, E0)
            assert U == U0 and B == B0
        assert sum(ranks[r][case][5] for r in range(world)) == phi0.size


def _dist_worker(rank, world, port, outdir):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    for p in (here, os.path.dirname(here)):
        if p not in sys.path:
            sys.path.insert(0, p)
    import numpy as np
    from _oracle_engine import MirrorDistEngine
    from paper_2101_07088_b200.geometry import ChargeSystem, SlabGeometry
    from paper_2101_07088_b200.params import plan_grid
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port,
                            rank=rank, world_size=world)
    try:
        geo = SlabGeometry(2.0, 2.0, 1.0, 1.0, 0.05, 1.0)
        system = ChargeSystem(geo, np.array([[0.5, 0.5, 0.5], [1.0, 1.0, 0.5]]),
                              np.array([1.0, -1.0]), 0.02)
        params = plan_grid(geo, 0.02, 1e-4, Nxy=64)
        eng = MirrorDistEngine()
        solver = ShardedSlabSolver(system, params, engine=eng, decompose=True)
        solver.solve_shard(eng.positions(system.positions))
        got = solver.buf["fields"].numpy().reshape(eng.Nz_pad, 4, eng.NXY)[:eng.Nz]
        ok = bool(np.allclose(got, eng.expected_fields(), rtol=0, atol=1e-12))
        with open(os.path.join(outdir, "dist%d.txt" % rank), "w") as f:
            f.write("ok" if ok else "mismatch")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_grid_pipeline_plumbing(tmp_path, world):
    """reduce-scatter -> all-to-all -> all-to-all -> all-reduce -> all-gather
    over gloo with the library's buffer layouts: every rank ends with the
    field grid of the summed spread grids."""
    if not hasattr(dist, "reduce_scatter_tensor"):
        pytest.skip("torch.distributed without reduce_scatter_tensor")
    mp.spawn(_dist_worker, args=(world, _free_port(), str(tmp_path)),
             nprocs=world, join=True)
    for r in range(world):
        assert (tmp_path / ("dist%d.txt" % r)).read_text() == "ok"


def _fault_worker(rank, world, port, outdir):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    for p in (here, os.path.dirname(here)):
        if p not in sys.path:
            sys.path.insert(0, p)
    from _oracle_engine import OracleShardEngine
    from test_oracle_golden import variant_problem

    class FaultyEngine(OracleShardEngine):
        """Rank 1 finds a charge of its own shard outside the z domain in
        its charge phase (the library reports FLAG_Z_OUTSIDE there)."""
        def charges(self, pos_all, count, need_forces):
            if dist.get_rank() == 1:
                raise ValueError("point outside the extended z domain")
            return super().charges(pos_all, count, need_forces)

    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port,
                            rank=rank, world_size=world)
    try:
        system, params, kw = variant_problem("c2n256")
        solver = ShardedSlabSolver(system, params,
                                   engine=FaultyEngine(system, params))
        try:
            solver.solve()
            res = "no error"
        except ValueError as exc:
            res = "ValueError: %s" % exc
        with open(os.path.join(outdir, "fault%d.txt" % rank), "w") as f:
            f.write(res)
    finally:
        dist.destroy_process_group()


def test_sharded_error_on_one_rank_raises_everywhere(tmp_path):
    """An error seen by one rank only is raised, with the same exception
    type, on every rank instead of leaving the others in a collective."""
    world = 3
    mp.spawn(_fault_worker, args=(world, _free_port(), str(tmp_path)),
             nprocs=world, join=True, daemon=False)
    for r in range(world):
        txt = (tmp_path / ("fault%d.txt" % r)).read_text()
        assert txt.startswith("ValueError"), (r, txt)
    assert "outside the extended z domain" in (tmp_path / "fault1.txt").read_text()
    assert "rank 1" in (tmp_path / "fault0.txt").read_text()


def test_cell_destinations_cover_every_neighbour():
    """Every charge is a target on exactly one rank, and every charge within
    r_cut (periodic in x) of a target is among that rank's sources."""
    import torch
    from paper_2101_07088_b200.sharded import cell_destinations
    rng = np.random.default_rng(5)
    L, halo = 2.0, 0.3
    x = rng.uniform(0, L, 4000)
    x[:4] = [0.0, L - 1e-12, 0.5 * L, 0.3]        # faces and exact boundaries
    for world in (1, 2, 3, 6):
        ci, dest, tgt = cell_destinations(torch.from_numpy(x), L, world, halo)
        ci, dest, tgt = ci.numpy(), dest.numpy(), tgt.numpy()
        assert np.array_equal(np.sort(ci[tgt]), np.arange(x.size))
        pairs = set(zip(ci.tolist(), dest.tolist()))
        assert len(pairs) == ci.size                  # never twice to a rank
        owner = dict(zip(ci[tgt].tolist(), dest[tgt].tolist()))
        sample = rng.choice(x.size, 300, replace=False)
        for i in sample:
            d = np.abs(x - x[i])
            d = np.minimum(d, L - d)
            for j in np.nonzero(d <= halo)[0]:
                assert (int(j), owner[int(i)]) in pairs
