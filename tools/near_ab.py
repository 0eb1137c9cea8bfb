"""A/B of near-field variants on one workload: stage timings with the
library's CUDA events (median of reps), each variant in a fresh process
(env switches are read once)."""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, json, numpy as np
sys.path.insert(0, %r)
from paper_2101_07088_b200 import workloads as W
from paper_2101_07088_b200.slab import SlabSolver
s, p = W.build(%r, N=%s)
sv = SlabSolver(s, p, precision=%r)
ts = []
for _ in range(%d):
    r = sv.solve(timings=True)
    ts.append(r.diagnostics["timings_ms"])
med = {k: float(np.median([t[k] for t in ts[1:]])) for k in ts[0]}
print("RESULT", json.dumps({"t": med, "U": r.U, "pairs": r.diagnostics["n_pairs"]}))
'''


def run(name, N, env, prec="fp64", reps=6):
    code = CODE % (REPO, name, N, prec, reps)
    out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env),
                         capture_output=True, text=True)
    for line in out.stdout.splitlines():
        if line.startswith("RESULT"):
            return json.loads(line[7:])
    return {"error": out.stderr[-1500:]}


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    N = sys.argv[2] if len(sys.argv) > 2 else "None"
    variants = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {"new": {}, "lists": {"SE_NEAR_LISTS": "1"}}
    prec = sys.argv[4] if len(sys.argv) > 4 else "fp64"
    res = {k: run(name, N, v, prec) for k, v in variants.items()}
    print(json.dumps(res, indent=1))
