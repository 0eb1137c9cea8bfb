"""Accuracy-check goldens from the REFERENCE package (build container):

    python tests/golden/make_checks.py

The reference's validate suites `xi` (xi-independence against the
no-splitting solve, validate.py:140-170, PAPER Table 3; 3 repetitions here
instead of 10) and `workcheck` (energy-force consistency, validate.py:175-
203, PAPER Table 5).  Stored in checks.npz next to this script.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from slabewald import validate as v                        # noqa: E402


def main():
    xi = v.check_xi_independence(reps=3)
    wc = v.check_workcheck()
    out = {"xi_values": np.array(v.XI_VALUES), "xi_std": np.array([r.value for r in xi]),
           "wc_reldiff": np.array([r.value for r in wc]),
           "wc_W1": np.array([r.detail["W1"] for r in wc]),
           "wc_W2": np.array([r.detail["W2"] for r in wc])}
    np.savez_compressed(os.path.join(HERE, "checks.npz"), **out)
    print(out)


if __name__ == "__main__":
    main()
