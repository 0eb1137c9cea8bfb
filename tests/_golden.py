"""Helpers to read the reference-generated fixtures (tests/golden)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def solves():
    raw = np.load(os.path.join(GOLDEN, "solves.npz"))
    out = {}
    for key in raw.files:
        case, field = key.split("__", 1)
        out.setdefault(case, {})[field] = raw[key]
    return out


def stages():
    return dict(np.load(os.path.join(GOLDEN, "stages_tiny.npz")))


def primitives():
    return dict(np.load(os.path.join(GOLDEN, "primitives.npz")))


def plans():
    with open(os.path.join(GOLDEN, "params.json")) as fh:
        return json.load(fh)


def rel_l2(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))
