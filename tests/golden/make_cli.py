"""CLI goldens from the REFERENCE package (build container):

    python tests/golden/make_cli.py

Runs the reference command line (slabewald/cli.py) on small configurations
and stores its outputs under tests/golden/cli/: ``tune`` reports and exit
codes, ``solve`` results.csv / summary.json, and a 2-step ``bd`` run
(trajectory.csv, density.csv, final_positions.npy).
"""

import contextlib
import io
import json
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "cli")
sys.path.insert(0, "/root/reference/pkg/src")

from slabewald import cli                                   # noqa: E402
from slabewald.geometry import save_charges_csv             # noqa: E402

CONF = """# C2-like box, bottom wall, open top
geometry.Lx = 2.0
geometry.Ly = 2.0
geometry.H = 1.0
geometry.eps_b = 0.05
geometry.eps_t = 1.0
g_w = 0.02
accuracy.delta = 1e-4
grid.Nxy = 64
"""
BD = """steric.a = 0.01
bd.dt = 1e-6
bd.steps = 2
bd.sample_every = 1
seed = 3
"""


def run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(io.StringIO()):
        code = cli.main(argv)
    return code, buf.getvalue()


def main():
    shutil.rmtree(OUT, ignore_errors=True)
    os.makedirs(OUT)
    rng = np.random.default_rng(7)
    n = 256
    pos = np.column_stack([rng.uniform(0, 2, n), rng.uniform(0, 2, n),
                           rng.uniform(0.12, 0.88, n)])
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    save_charges_csv(os.path.join(OUT, "charges.csv"), pos, q)
    with open(os.path.join(OUT, "solve.conf"), "w") as fh:
        fh.write(CONF)
    with open(os.path.join(OUT, "bd.conf"), "w") as fh:
        fh.write(CONF + BD)
    with open(os.path.join(OUT, "bad.conf"), "w") as fh:
        fh.write(CONF + "grid.xi = 3.0\n")
    with open(os.path.join(OUT, "tight.conf"), "w") as fh:
        fh.write(CONF.replace("grid.Nxy = 64", "grid.Nxy = 8"))
    codes = {}
    for name in ("solve", "tight", "bad"):
        code, text = run(["tune", "--config", os.path.join(OUT, name + ".conf")])
        codes["tune_" + name] = code
        if code in (0, 3):
            with open(os.path.join(OUT, "tune_%s.json" % name), "w") as fh:
                fh.write(text)
    codes["solve"], _ = run(["solve", "--config", os.path.join(OUT, "solve.conf"),
                             "--charges", os.path.join(OUT, "charges.csv"),
                             "--out", os.path.join(OUT, "ref_solve")])
    codes["bd"], _ = run(["bd", "--config", os.path.join(OUT, "bd.conf"),
                          "--charges", os.path.join(OUT, "charges.csv"),
                          "--out", os.path.join(OUT, "ref_bd")])
    codes["missing_charges"], _ = run(["solve", "--config", os.path.join(OUT, "solve.conf")])
    with open(os.path.join(OUT, "codes.json"), "w") as fh:
        json.dump(codes, fh, indent=1, sort_keys=True)
    print(codes)


if __name__ == "__main__":
    main()
