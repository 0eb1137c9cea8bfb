"""Stage-by-stage comparison of the GPU path with the oracle (prints errors
instead of asserting; used while bringing up kernels on the GPU box)."""
import os
import sys
import time
import traceback

os.environ.setdefault("SE_KEEP_STAGES", "1")
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

import numpy as np

from oracle import slab_oracle as O
from paper_2101_07088_b200 import workloads as W
from paper_2101_07088_b200.geometry import ChargeSystem, SlabGeometry
from paper_2101_07088_b200.params import plan_grid
from paper_2101_07088_b200.slab import SlabSolver
from _golden import rel_l2, stages


def report(name, a, b):
    print("  %-12s rel_l2 %.3e  (|ref| %.3e)" % (name, rel_l2(a, b),
                                               np.linalg.norm(b)))


def stage_case(system, params, label):
    print("==", label, "grid", params.Nx, params.Ny, params.Nz, "N", system.n)
    t = time.time()
    solver = SlabSolver(system, params)
    res = solver.solve(timings=True)
    print("  gpu solve %.3fs (incl. first-call)" % (time.time() - t))
    cap = {}
    ref = O.OracleSlabSolver(system, params).solve(capture=cap)
    nx, ny, nz = params.Nx, params.Ny, params.Nz
    nyh = ny // 2 + 1
    rho = solver.debug_fetch(0).reshape(nz, 2, nx, ny).transpose(1, 2, 3, 0)
    if "rho_over" in cap:
        report("rho_over", rho[0], cap["rho_over"])
    report("rho_in", rho[1], cap["rho_in"])
    keep = solver.debug_fetch(1).view(np.complex128).reshape(nz, 2, nx, nyh)
    psi = keep.transpose(1, 2, 3, 0)
    if cap.get("psi_o") is not None:
        report("psi_o", psi[0], cap["psi_o"][:, :nyh])
    report("psi_i", psi[1], cap["psi_i"][:, :nyh])
    if cap.get("mismatch") is not None:
        mism = solver.debug_fetch(3).view(np.complex128).reshape(4, nx, nyh)
        for i, key in enumerate(("phi_b", "e_b", "phi_t", "e_t")):
            report("m_" + key, mism[i], cap["mismatch"][key][:, :nyh])
    fields = solver.debug_fetch(2).reshape(nz, 4, nx, ny).transpose(1, 2, 3, 0)
    A_i = cap["k0"]["A_i"]
    print("  A_i gpu %.15e ref %.15e" % (res.diagnostics["k0"].A_i, A_i))
    z = O.cheb_nodes(nz, params.z0, params.z1)
    rf = cap["fields"]
    report("psi grid", fields[0] + A_i * z, rf[0])
    report("Ex grid", -fields[1], rf[1])
    report("Ey grid", -fields[2], rf[2])
    report("Ez grid", -(fields[3] + A_i), rf[3])
    far = solver.debug_fetch(4).reshape(4, -1)
    cell = solver.grid.hx * solver.grid.hy
    report("phi_far", cell * far[0], cap["phi_far"])
    near = solver.debug_fetch(5).reshape(4, -1)
    report("phi_near", near[0], cap["phi_near"])
    if cap.get("e_near") is not None:
        report("E_near", near[1:4].T, cap["e_near"])
    phi, E, U, diag = ref
    report("phi_bar", res.phi_bar, phi)
    report("E_bar", res.E_bar, E)
    print("  U gpu %.15e ref %.15e  B_i %.6e vs %.6e" % (res.U, U,
          res.diagnostics["B_i"], diag["B_i"]))
    print("  pairs", res.diagnostics["n_pairs"], "launches",
          res.diagnostics["n_launches"], "timings", res.diagnostics.get("timings_ms"))


def main():
    g = stages()
    geo = SlabGeometry(1.5, 1.5, 1.0, 1.0, 0.05, 0.02)
    system = ChargeSystem(geo, g["positions"], g["charges"], 0.03)
    params = plan_grid(geo, 0.03, 1e-4, Nxy=24)
    for label, (s, p) in [("tiny", (system, params)),
                          ("c1", W.build("c1")),
                          ("c2", W.build("c2")),
                          ("c3n4096", W.build("c3", N=4096))]:
        try:
            stage_case(s, p, label)
        except Exception:
            traceback.print_exc()
    # timing of C4 (no oracle)
    try:
        s, p = W.build("c4")
        solver = SlabSolver(s, p)
        for it in range(3):
            t = time.time()
            res = solver.solve(timings=True)
            print("c4 solve %.4fs" % (time.time() - t), res.diagnostics["timings_ms"],
                  "pairs", res.diagnostics["n_pairs"], "U", res.U)
    except Exception:
        traceback.print_exc()


if __name__ == "__main__":
    main()
