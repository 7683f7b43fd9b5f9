"""The command line against the reference CLI (cli.py), run by tests/golden/make_golden.py.

Every case compares the exit code, stdout, stderr and every file written with what
the unmodified reference printed and wrote for the same argv. ``time_ms`` is the one
wall-clock column in the bench CSV and is left out of that comparison. The CPU test
runs the cases that never reach the solver: generate, usage, parse and config errors.
The GPU test runs all of them.
"""

import contextlib
import io
import os

import numpy as np
import pytest

from conftest import rel_err

from paper_2203_05027_b200.cli import run_cli

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "cli_cases.npz")


def _close(got, want):
    """Texts equal token by token; numeric tokens to 1e-9 relative. The reports' dot
    products (pobj, dobj, gap, 2-norms) are BLAS np.dot in the reference and a fixed-order
    device reduction here, so they agree to rounding."""
    gl, wl = got.splitlines(), want.splitlines()
    if len(gl) != len(wl):
        return False
    for g, w in zip(gl, wl):
        gt, wt = g.replace(",", " ").split(), w.replace(",", " ").split()
        if len(gt) != len(wt):
            return False
        for a, b in zip(gt, wt):
            if a == b:
                continue
            try:
                fa, fb = float(a), float(b)
            except ValueError:
                return False
            if not abs(fa - fb) <= 1e-9 * max(1.0, abs(fb)):
                return False
    return True


def _solution_vectors(text):
    return np.array([float(v) for v in text.splitlines()[2:]])


def _strip_time(csv_text):
    lines = csv_text.splitlines()
    col = lines[0].split(",").index("time_ms")
    return [[c for k, c in enumerate(line.split(",")) if k != col] for line in lines]


def _run_cases(d, with_gpu):
    z = np.load(GOLDEN)
    with open(os.path.join(d, "bad.txt"), "w") as f:
        f.write("CONEPROB 1\n2 2 1\nCONES 1 2\n0 5 1.0\n1.0\n2.0\n1.0\n1.0\n")
    files = {}
    for c, name, text in zip(z["file_case"], z["file_name"], z["file_text"]):
        files.setdefault(int(c), {})[str(name)] = str(text)
    ran = 0
    for i, argv in enumerate(z["argv"]):
        if bool(z["gpu"][i]) and not with_gpu:
            continue
        before = set(os.listdir(d))
        so, se = io.StringIO(), io.StringIO()
        with contextlib.redirect_stdout(so), contextlib.redirect_stderr(se):
            rc = run_cli(str(argv).replace("{d}", str(d)).split())
        assert rc == int(z["rc"][i]), argv
        assert _close(so.getvalue().replace(str(d), "{d}"), str(z["stdout"][i])), argv
        assert se.getvalue().replace(str(d), "{d}") == str(z["stderr"][i]), argv
        written = sorted(set(os.listdir(d)) - before)
        want = files.get(i, {})
        assert written == sorted(want), argv
        for name in written:
            with open(os.path.join(d, name), encoding="utf-8") as f:
                got = f.read()
            if name.endswith(".csv") and "time_ms" in want[name].split("\n", 1)[0]:
                g, w = _strip_time(got), _strip_time(want[name])
                assert _close("\n".join(map(" ".join, g)), "\n".join(map(" ".join, w))), (argv, name)
            elif name.endswith(".sol"):
                # x then lam: the reduced iteration agrees with the literal one to rounding
                # (rel_err <= 1e-8 after a full solve, as test_gpu_parity's solves)
                assert got.splitlines()[0] == want[name].splitlines()[0], (argv, name)
                assert _close(got.splitlines()[1], want[name].splitlines()[1]), (argv, name)
                assert rel_err(_solution_vectors(got), _solution_vectors(want[name])) <= 1e-8, (argv, name)
            else:
                assert _close(got, want[name]), (argv, name)
                if name.endswith(".txt"):
                    assert got == want[name], (argv, name)
        ran += 1
    return ran


def test_cli_host_cases(tmp_path):
    assert _run_cases(tmp_path, with_gpu=False) >= 8


@pytest.mark.gpu
def test_cli_matches_reference(tmp_path):
    assert _run_cases(tmp_path, with_gpu=True) == len(np.load(GOLDEN)["argv"])
