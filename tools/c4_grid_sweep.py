"""C4 (N = 2^20, Lx = Ly = 2H, eps_b = eps_t = 0.05, delta = 1e-4) at
several transverse grid sizes: the near/far split of the Ewald sum is a free
parameter (plan_grid's N_xy sets xi, hence the near-field cutoff and the
number of pairs, against the grid size), and the reference/paper quote each
method at its own optimum N_xy.  Each grid is planned for the same delta by
plan_grid, so every point solves the same problem to the same tolerance; the
forces are compared against the N_xy = 256 solve (relative L2) to show it.

Device time per solve: CUDA events around the device-resident call, L2
flushed (256 MB write) before each step, median of ``steps`` after
``warmup``.  Per-stage times come from one extra solve with the library's
stage timers.

    python tools/c4_grid_sweep.py [steps] [Nxy ...]
"""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2101_07088_b200 import workloads as W                # noqa: E402
from paper_2101_07088_b200.slab import SlabSolver               # noqa: E402

SWEEP = (256, 288, 320, 352)


def measure(steps=10, warmup=3, sweep=SWEEP, name="c4"):
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = {"workload": name, "timing": "CUDA events, L2 flushed, median", "points": {}}
    E_ref = None
    for nxy in sweep:
        system, params = W.build(name, Nxy=nxy)
        n = system.n
        pos = torch.as_tensor(system.positions, device=dev).contiguous()
        phi = torch.empty(n, dtype=torch.float64, device=dev)
        E = torch.empty((n, 3), dtype=torch.float64, device=dev)
        s = SlabSolver(system, params, device=0)
        s.set_stream(stream.cuda_stream)
        for _ in range(warmup):
            s.solve_device(pos.data_ptr(), phi.data_ptr(), E.data_ptr(), n)
        torch.cuda.synchronize()
        times = []
        for _ in range(steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _, diag = s.solve_device(pos.data_ptr(), phi.data_ptr(), E.data_ptr(), n)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        flush.zero_()
        _, dt = s.solve_device(pos.data_ptr(), phi.data_ptr(), E.data_ptr(), n,
                               timings=True)
        torch.cuda.synchronize()
        Eh = E.cpu().numpy()
        if E_ref is None:
            E_ref = Eh
        rel = float(np.linalg.norm(Eh - E_ref) / np.linalg.norm(E_ref))
        ms = float(np.median(times))
        out["points"][str(nxy)] = {
            "grid": [params.Nx, params.Ny, params.Nz], "xi": params.xi,
            "r_cut": params.r_cut, "ms": ms, "charges_per_s": n / (ms * 1e-3),
            "pairs": int(diag.n_pairs),
            "stage_ms": [round(float(x), 4) for x in dt.t_ms[8:14]],
            "E_rel_l2_vs_%d" % sweep[0]: rel}
        s.close()
        del pos, phi, E
        torch.cuda.empty_cache()
    best = min(out["points"].items(), key=lambda kv: kv[1]["ms"])
    out["opt"] = {"Nxy": int(best[0]), "ms": best[1]["ms"]}
    out["stage_ms_keys"] = "t_ms[8:14] (k_spread, k_bvp, k_interp, k_near, k_near_scan, k_near_eval)"
    return out


if __name__ == "__main__":
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    sweep = tuple(int(x) for x in sys.argv[2:]) or SWEEP
    print(json.dumps(measure(steps=steps, sweep=sweep)))
