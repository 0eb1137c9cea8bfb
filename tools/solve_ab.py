"""A/B of whole-solve variants selected by environment switches: device
time of a full solve (CUDA events on the solver's stream, L2 flushed between
solves outside the event pair, median of reps), each variant in a fresh
process (the switches are read once).

    python tools/solve_ab.py c4 '{"serial": {}, "fork2": {"SE_NEAR_OVERLAP": "2"}}' [fp64|fp32] [graph]
"""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, %r)
from paper_2101_07088_b200 import workloads as W
from paper_2101_07088_b200.slab import SlabSolver
s, p = W.build(%r)
sv = SlabSolver(s, p, precision=%r)
st = torch.cuda.current_stream()
sv.set_stream(st.cuda_stream)
n = s.positions.shape[0]
pos = torch.tensor(np.ascontiguousarray(s.positions), dtype=torch.float64, device="cuda")
phi = torch.empty(n, dtype=torch.float64, device="cuda")
E = torch.empty((n, 3), dtype=torch.float64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
graph = %r
ts, Us = [], []
for it in range(%d):
    flush.fill_(it & 255)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    U, _ = sv.solve_device(pos.data_ptr(), phi.data_ptr(), E.data_ptr(), n, graph=graph)
    b.record(st)
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b)); Us.append(U)
print("RESULT", json.dumps({"ms": float(np.median(ts[3:])), "min": float(np.min(ts[3:])),
                            "U": Us[-1], "phi0": float(phi[0]), "E0": float(E[0, 0])}))
'''


def run(name, env, prec="fp64", graph=False, reps=15):
    code = CODE % (REPO, name, prec, graph, reps)
    out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env),
                         capture_output=True, text=True)
    for line in out.stdout.splitlines():
        if line.startswith("RESULT"):
            return json.loads(line[7:])
    return {"error": out.stderr[-1500:]}


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    variants = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {"serial": {}}
    prec = sys.argv[3] if len(sys.argv) > 3 else "fp64"
    graph = len(sys.argv) > 4 and sys.argv[4] == "graph"
    res = {k: run(name, v, prec, graph) for k, v in variants.items()}
    print(json.dumps(res, indent=1))
