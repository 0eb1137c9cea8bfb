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


_MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def mix64(s):
    """splitmix64 finaliser of source indices (uint64 wrap-around), the
    per-pair term of the order-independent pair-set hash that the library
    computes on the device (SE_PAIR_HASH, csrc/se_near.cu)."""
    with np.errstate(over="ignore"):
        z = np.asarray(s, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def pair_hash(e, s, n):
    """(count[n], hash[n]) of a pair list (target e, source s): the number
    of sources of each target and the wrap-around sum of mix64(source) --
    equal for two lists exactly when their pair SETS agree (up to a 2^-64
    collision chance per target)."""
    e = np.asarray(e, dtype=np.int64)
    cnt = np.bincount(e, minlength=n).astype(np.int64)
    h = np.zeros(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        np.add.at(h, e, mix64(s))
    return cnt, h
