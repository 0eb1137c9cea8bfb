"""A few triply periodic force evaluations at the paper configuration (for
ncu launch lists)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_07088_b200 import workloads as W
from paper_2101_07088_b200.periodic import TriplyPeriodicSolver
system, params = W.build("paper")
geo = system.geometry
tp = TriplyPeriodicSolver((geo.Lx, geo.Ly, 2 * geo.H), 70, system.g_w, geo.eps, delta=1e-4)
print("r_cut", tp.r_cut, "grid", tp.n, "radius", tp.radius)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    f = tp.forces(system.positions, system.charges)
print(abs(f).max())
