"""Device-resident BD steps at scale (BASELINE configs[4]: the C5 double
layer, forces every step) on ONE GPU: ms per BD step (solve with
need_energy=False + steric pair forces + the step kernel with its rejection
check), CUDA events on the solver's stream, after warm-up.

    python tools/bd_scale.py [c4|c5] [steps]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_07088_b200 import bd as B                 # noqa: E402
from paper_2101_07088_b200 import workloads as W          # noqa: E402
from paper_2101_07088_b200.slab import SlabSolver         # noqa: E402


def measure(name="c4", steps=10, warmup=3):
    system, params = W.build(name)
    geo = system.geometry
    zb = params.n_sigma * system.g_w
    start = system.positions.copy()
    pad = 0.02 * geo.H
    start[:, 2] = (zb + pad) + (start[:, 2] - zb) * (geo.H - 2 * zb - 2 * pad) / (geo.H - 2 * zb)
    steric = B.StericParams(a=0.5 * system.g_w)
    cfg = B.BdConfig(dt=1e-8, steps=steps, seed=1, max_disp=steric.a)
    solver = SlabSolver(system, params)
    bd = B.DeviceBd(solver, steric, cfg, positions=start)
    bd.step(warmup)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(bd.stream)
    bd.step(steps)
    e1.record(bd.stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / steps
    out = {"workload": name, "N": int(system.charges.size),
           "grid": [params.Nx, params.Ny, params.Nz], "ms_per_bd_step": ms,
           "charges_per_s": system.charges.size / (ms * 1e-3),
           "rejections": int(bd.rejections.value), "steps": steps}
    solver.close()
    return out


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    print(json.dumps(measure(name, int(sys.argv[2]) if len(sys.argv) > 2 else 10)))
