"""Command line against the reference CLI's own
outputs (tests/golden/make_cli.py): tune reports and exit codes on CPU,
solve / bd output files on the GPU."""

import contextlib
import io
import json
import os

import numpy as np
import pytest

from paper_2101_07088_b200 import cli

G = os.path.join(os.path.dirname(__file__), "golden", "cli")
CODES = json.load(open(os.path.join(G, "codes.json")))


def _run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(io.StringIO()):
        code = cli.main(argv)
    return code, buf.getvalue()


@pytest.mark.parametrize("name", ["solve", "tight", "bad"])
def test_tune_matches_reference(name):
    code, text = _run(["tune", "--config", os.path.join(G, name + ".conf")])
    assert code == CODES["tune_" + name]
    ref = os.path.join(G, "tune_%s.json" % name)
    if os.path.exists(ref):
        assert json.loads(text) == json.load(open(ref))


def test_config_errors_exit_codes(tmp_path):
    assert _run(["solve", "--config", os.path.join(G, "solve.conf")])[0] == \
        CODES["missing_charges"]
    bad = tmp_path / "x.conf"
    bad.write_text("geometry.Lx 2.0\n")
    assert _run(["tune", "--config", str(bad)])[0] == cli.EXIT_CONFIG
    assert _run(["validate"])[0] == cli.EXIT_CONFIG


def _csv(path):
    lines = open(path).read().splitlines()
    return lines[0], np.array([[float(v) for v in ln.split(",")] for ln in lines[1:]])


@pytest.mark.gpu
def test_gpu_solve_outputs_match_reference(tmp_path):
    code, _ = _run(["solve", "--config", os.path.join(G, "solve.conf"),
                    "--charges", os.path.join(G, "charges.csv"), "--out", str(tmp_path)])
    assert code == 0
    h, got = _csv(tmp_path / "results.csv")
    h0, ref = _csv(os.path.join(G, "ref_solve", "results.csv"))
    assert h == h0 and got.shape == ref.shape
    assert np.array_equal(got[:, 0], ref[:, 0])
    for cols in ((1,), (2, 3, 4), (5, 6, 7)):
        c = list(cols)
        assert np.linalg.norm(got[:, c] - ref[:, c]) <= 1e-10 * np.linalg.norm(ref[:, c])
    s, s0 = json.load(open(tmp_path / "summary.json")), \
        json.load(open(os.path.join(G, "ref_solve", "summary.json")))
    assert s["params"] == s0["params"]
    assert abs(s["U"] - s0["U"]) <= 1e-10 * abs(s0["U"])
    assert abs(s["B_i"] - s0["B_i"]) <= 1e-9 * max(abs(s0["B_i"]), 1.0)


@pytest.mark.gpu
def test_gpu_bd_outputs_match_reference(tmp_path):
    code, _ = _run(["bd", "--config", os.path.join(G, "bd.conf"),
                    "--charges", os.path.join(G, "charges.csv"), "--out", str(tmp_path)])
    assert code == 0
    pos = np.load(tmp_path / "final_positions.npy")
    pos0 = np.load(os.path.join(G, "ref_bd", "final_positions.npy"))
    assert np.max(np.abs(pos - pos0)) < 1e-10
    h, d = _csv(tmp_path / "density.csv")
    h0, d0 = _csv(os.path.join(G, "ref_bd", "density.csv"))
    assert h == h0 and np.array_equal(d, d0)
    h, t = _csv(tmp_path / "trajectory.csv")
    h0, t0 = _csv(os.path.join(G, "ref_bd", "trajectory.csv"))
    assert h == h0 and np.array_equal(t[:, :2], t0[:, :2])
    assert np.allclose(t[:, 2], t0[:, 2], rtol=1e-9, atol=0)
