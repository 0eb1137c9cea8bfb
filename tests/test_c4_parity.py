"""Parity at the north-star grid and density (VERDICT r01 "next" #1).

Goldens: tests/golden/c4.npz, made by RUNNING THE REFERENCE
(tests/golden/make_c4.py):
  * c4n64k -- the C4 box and grid (256 x 256 x 258, Nz = 258 so the even /
    odd DCT fold at 129 + 129 is exercised), N = 65536;
  * c4d -- C4 density and spacing (L = 0.5, 64 x 64 x 258, ~600 near pairs
    per charge: the large-N near-field path), N = 65536, with the
    reference's pair SET (NearField._pairs) as per-charge counts and
    order-independent hashes.
fp64: phi, E, U within 1e-10 relative L2 and the pair set exactly equal.
fp32 mode: within the run's Ewald tolerance (delta = 1e-4) -- asserted at
delta / 10 -- and the same exact pair set (membership is the fp64 test).
"""
import os

import numpy as np
import pytest

from paper_2101_07088_b200 import workloads as W
from _golden import GOLDEN, pair_hash, rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-10
DELTA = 1e-4


def _gold(case):
    raw = np.load(os.path.join(GOLDEN, "c4.npz"))
    return {k.split("__", 1)[1]: raw[k] for k in raw.files if k.startswith(case + "__")}


def _check(res, g, tol):
    assert rel_l2(res.phi_bar, g["phi"]) < tol, rel_l2(res.phi_bar, g["phi"])
    assert rel_l2(res.E_bar, g["E"]) < tol, rel_l2(res.E_bar, g["E"])
    U = float(g["U"])
    assert abs(res.U - U) <= tol * max(1.0, abs(U)), (res.U, U)
    B = float(g["B_i"])
    assert abs(res.diagnostics["B_i"] - B) <= tol * max(1.0, abs(B))


@pytest.mark.parametrize("case,name", [("c4n64k", "c4"), ("c4d", "c4d")])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_c4_against_reference(case, name, precision):
    from paper_2101_07088_b200.slab import SlabSolver
    g = _gold(case)
    system, params = W.build(name, N=65536)
    solver = SlabSolver(system, params, precision=precision)
    res = solver.solve(record_pairs=(case == "c4d"))
    _check(res, g, TOL if precision == "fp64" else 0.1 * DELTA)
    if case == "c4d":
        cnt, h = solver.pair_set()
        assert int(cnt.sum()) == int(g["n_pairs"])
        assert np.array_equal(cnt, g["pair_count"].astype(np.int64))
        assert np.array_equal(h, g["pair_hash"])
        assert res.diagnostics["n_pairs"] == int(g["n_pairs"])
    solver.close()


def test_pair_set_small_case_exact():
    """The N = 512 C2 case (fused one-warp-per-point near-field path): the
    device pair set equals the reference's stored pair list."""
    from paper_2101_07088_b200.slab import SlabSolver
    gp = np.load(os.path.join(GOLDEN, "pairs_c2n512.npz"))
    system, params = W.build("c2", N=512)
    solver = SlabSolver(system, params)
    solver.solve(record_pairs=True)
    cnt, h = solver.pair_set()
    rc, rh = pair_hash(gp["e"], gp["s"], 512)
    assert np.array_equal(cnt, rc)
    assert np.array_equal(h, rh)
    solver.close()


@pytest.mark.parametrize("env", [{"SE_NEAR_FUSED": "0"}, {"SE_NEAR_FUSED": "1"},
                                 {"SE_NEAR_FUSED": "0", "SE_NEAR_LIST_SCALE": "0.3"}])
def test_pair_set_all_paths_c4d(env):
    """Every near-field path gives the reference's pair set: scan -> lists
    -> eval (default at this size), one warp per point (SE_NEAR_FUSED=1),
    and the list path with capacities
    cut so that points overflow into the fallback kernel."""
    import subprocess
    import sys
    code = (
        "import numpy as np, sys; sys.path.insert(0, 'tests');"
        "from paper_2101_07088_b200 import workloads as W;"
        "from paper_2101_07088_b200.slab import SlabSolver;"
        "from _golden import GOLDEN;"
        "raw = np.load(GOLDEN + '/c4.npz');"
        "s, p = W.build('c4d', N=65536); sv = SlabSolver(s, p);"
        "sv.solve(record_pairs=True); c, h = sv.pair_set();"
        "assert np.array_equal(h, raw['c4d__pair_hash']);"
        "assert np.array_equal(c, raw['c4d__pair_count'].astype(np.int64));"
        "print('ok')")
    env = dict(os.environ, **env)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("mode", ["0", "1", "2", "3"])
def test_near_fork_modes_c4d(mode):
    """The near-field stream fork (SE_NEAR_OVERLAP: 0 serial, 1 whole near
    field on the side stream, 2 its scan only -- the default, 3 the grid
    pipeline on the side stream) gives the reference's results and pair set,
    eagerly and as a replayed CUDA graph, and every mode gives the same
    device results bit for bit."""
    import subprocess
    import sys
    code = (
        "import numpy as np, sys, torch, hashlib; sys.path.insert(0, 'tests');"
        "from paper_2101_07088_b200 import workloads as W;"
        "from paper_2101_07088_b200.slab import SlabSolver;"
        "from _golden import GOLDEN, rel_l2;"
        "raw = np.load(GOLDEN + '/c4.npz');"
        "s, p = W.build('c4d', N=65536); sv = SlabSolver(s, p);"
        "r = sv.solve(record_pairs=True); c, h = sv.pair_set();"
        "assert np.array_equal(h, raw['c4d__pair_hash']);"
        "assert rel_l2(r.phi_bar, raw['c4d__phi']) < 1e-10;"
        "assert rel_l2(r.E_bar, raw['c4d__E']) < 1e-10;"
        "n = s.n; st = torch.cuda.current_stream(); sv.set_stream(st.cuda_stream);"
        "pos = torch.tensor(s.positions, device='cuda');"
        "phi = torch.empty(n, dtype=torch.float64, device='cuda');"
        "E = torch.empty((n, 3), dtype=torch.float64, device='cuda');"
        "Us = [sv.solve_device(pos.data_ptr(), phi.data_ptr(), E.data_ptr(), n, graph=True)[0]"
        "      for _ in range(4)];"
        "torch.cuda.synchronize();"
        "assert len(set(Us)) == 1, Us;"
        "assert rel_l2(phi.cpu().numpy(), raw['c4d__phi']) < 1e-10;"
        "dig = hashlib.sha1(phi.cpu().numpy().tobytes() + E.cpu().numpy().tobytes()).hexdigest();"
        "print('ok', dig)")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    digs = {}
    for m in sorted({mode, "2"}):
        env = dict(os.environ, SE_NEAR_OVERLAP=m)
        out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env,
                             capture_output=True, text=True, timeout=600)
        assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
        digs[m] = out.stdout.split()[-1]
    assert len(set(digs.values())) == 1, digs


def test_graph_replay_through_list_overflow_c4d():
    """Repeated host-API solves (CUDA-graph replay) with pair-list
    capacities cut so the lists overflow: each overflow runs the fallback
    kernel, doubles the capacities and retires the graph; the next solve
    runs eagerly and a later one is captured again -- every result equals
    the reference's."""
    import subprocess
    import sys
    code = (
        "import numpy as np, sys; sys.path.insert(0, 'tests');"
        "from paper_2101_07088_b200 import workloads as W;"
        "from paper_2101_07088_b200.slab import SlabSolver;"
        "from _golden import GOLDEN, rel_l2;"
        "raw = np.load(GOLDEN + '/c4.npz');"
        "s, p = W.build('c4d', N=65536); sv = SlabSolver(s, p);"
        "us = []\n"
        "for _ in range(7):\n"
        "    r = sv.solve()\n"
        "    assert rel_l2(r.phi_bar, raw['c4d__phi']) < 1e-10\n"
        "    assert rel_l2(r.E_bar, raw['c4d__E']) < 1e-10\n"
        "    assert r.diagnostics['n_pairs'] == int(raw['c4d__n_pairs'])\n"
        "    us.append(r.U)\n"
        "print('ok', len(set(us)))")
    env = dict(os.environ, SE_NEAR_LIST_SCALE="0.2")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_fp32_graph_replay_c4():
    """fp32 mode through repeated host-API solves (warm, capture, replay)
    at the C4 grid: every result within delta / 10 of the reference's."""
    from paper_2101_07088_b200.slab import SlabSolver
    g = _gold("c4n64k")
    system, params = W.build("c4", N=65536)
    solver = SlabSolver(system, params, precision="fp32")
    for _ in range(3):
        _check(solver.solve(), g, 0.1 * DELTA)
    solver.close()
