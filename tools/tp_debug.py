"""Debug helper: one call of each triply periodic entry point."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_07088_b200 import bd as B
from paper_2101_07088_b200.periodic import TriplyPeriodicSolver
G = np.load("tests/golden/tp.npz")
box = float(G["g2_box"]); boxes = (box, box, box)
which = sys.argv[1]
if which == "steric":
    st = B.StericParams(a=1.0, U0=0.2233, r_m=1.0, p=2)
    f = B.steric_pair_forces(G["g2_pos"], st, boxes)
    print("steric", np.abs(f - G["g2_steric"]).max())
else:
    s = TriplyPeriodicSolver(boxes, 32, 0.25, float(G["g2_eps"]), delta=5e-4)
    f = s.forces(G["g2_pos"], G["g2_q"])
    print("tp", np.abs(f - G["g2_forces"]).max())
