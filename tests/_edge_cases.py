"""Edge-case inputs shared by the golden generator and the parity tests
(tests/golden/make_edges.py, tests/test_edges.py): small systems on the C2 box (L = 2, H = 1,
eps_b = 0.05, eps_t = 1, g_w = 0.02, delta = 1e-4, 64 x 64 xy modes)."""

import numpy as np

L, H, G_W, DELTA, NXY = 2.0, 1.0, 0.02, 1e-4, 64
GEO = (L, L, H, 1.0, 0.05, 1.0)


def _random(n, seed):
    rng = np.random.default_rng(seed)
    pos = np.column_stack([rng.uniform(0, L, n), rng.uniform(0, L, n),
                           rng.uniform(0.1, 0.9, n)])
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    return pos, q


def _coincident():
    pos, q = _random(64, 21)
    pos[1] = pos[0]                     # +1 / -1 at the same point
    pos[5] = pos[4]
    pos[9] = pos[8]
    return pos, q


def _on_nodes():
    pos, q = _random(64, 22)
    h = L / NXY
    pos[:16, 0] = h * np.arange(16) * 3
    pos[:16, 1] = h * np.arange(16) * 2
    return pos, q


def _at_cutoff():
    from paper_2101_07088_b200.params import plan_grid
    from paper_2101_07088_b200.geometry import SlabGeometry
    p = plan_grid(SlabGeometry(*GEO), G_W, DELTA, Nxy=NXY)
    pos, q = _random(64, 23)
    pos[0] = [0.5, 0.5, 0.5]
    pos[1] = [0.5 + p.r_cut, 0.5, 0.5]
    pos[2] = [1.0, 1.0, 0.4]
    pos[3] = [1.0, 1.0, 0.4 + p.r_cut]
    return pos, q


def _walls():
    pos, q = _random(64, 24)
    pos[:4, 2] = [0.0, 0.0, H, H]
    return pos, q


def _periodic_edge():
    pos, q = _random(64, 25)
    pos[0, 0] = 0.0
    pos[1, 0] = np.nextafter(L, 0.0)
    pos[2, 1] = 0.0
    pos[3, 1] = np.nextafter(L, 0.0)
    pos[4, :2] = [np.nextafter(L, 0.0), np.nextafter(L, 0.0)]
    return pos, q


def _single():
    return np.array([[1.0, 1.0, 0.5]]), np.array([1.0])


def _empty():
    return np.zeros((0, 3)), np.zeros(0)


CASES = {"coincident": _coincident, "on_nodes": _on_nodes,
         "at_cutoff": _at_cutoff, "walls": _walls,
         "periodic_edge": _periodic_edge, "single": _single,
         "empty": _empty}


def build(name):
    """(geometry args, positions, charges, g_w, delta, Nxy) of a case."""
    pos, q = CASES[name]()
    return GEO, pos, q, G_W, DELTA, NXY
