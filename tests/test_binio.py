"""CONEPROB reader/writer (csrc/cf_io.cpp via binio.py) and the binary format — host only.

Golden: tests/golden/coneprob_cases.npz holds, for valid and malformed texts,
the unmodified reference's parse_problem outcome (fileio.py:98-190): the
ParseError line and message, another exception, or a hash of the parsed arrays.
"""

import hashlib
import os

import numpy as np
import pytest

from conftest import load_golden
from paper_2203_05027_b200 import binio
from paper_2203_05027_b200.instances import GenSpec, generate


def _sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _outcome(fn, text):
    try:
        p = fn(text)
        return (-1, "", _sha(p.A.rows, p.A.cols, p.A.vals, p.b, p.c, np.asarray(p.cones.block_sizes)))
    except binio.ParseError as e:
        return (e.line, e.message, "")
    except Exception as e:
        return (-2, f"{type(e).__name__}: {e}", "")


@pytest.mark.parametrize("fn", ["native", "python"])
def test_parse_matches_reference_outcomes(fn):
    g = load_golden("coneprob_cases.npz")
    parse = binio.parse_problem if fn == "native" else binio._parse_problem_py
    for k, text in enumerate(g["texts"]):
        want = (int(g["lines"][k]), str(g["messages"][k]), str(g["hashes"][k]))
        assert _outcome(parse, str(text)) == want, (k, repr(str(text))[:120])


def test_write_reproduces_reference_text():
    g = load_golden("coneprob_cases.npz")
    base = str(g["texts"][0])           # written by the reference's write_problem
    assert binio.write_problem(binio.parse_problem(base)) == base


def test_format_float_is_python_repr():
    rng = np.random.default_rng(0)
    vals = np.concatenate([rng.standard_normal(2000), rng.standard_normal(500) * 10.0 ** rng.integers(-30, 30, 500),
                           [0.0, -0.0, 1.0, 1e16, 1e15, 123456789012345678.0, 1e-4, 1e-5, 0.1, 5e-324,
                            1.7976931348623157e308, float("inf"), -float("inf"), 100.0, 1e22, 2.5e-7]])
    for v in vals:
        assert binio.format_float(v) == repr(float(v)), v


def test_large_parse_multichunk_and_errors(tmp_path):
    """Many parser chunks: native == line-by-line restatement, including late errors and duplicates."""
    p = generate(GenSpec(300, 1200, 0.08, "lp", seed=11))   # ~28.8k entries
    text = binio.write_problem(p)
    path = tmp_path / "p.txt"
    path.write_text(text)
    q = binio.read_problem(str(path), threads=8)
    r = binio._parse_problem_py(text)
    for a, b in ((q.A.rows, r.A.rows), (q.A.cols, r.A.cols), (q.A.vals, r.A.vals), (q.b, r.b), (q.c, r.c)):
        assert np.array_equal(a, b)
    lines = text.splitlines()
    nnz = p.A.nnz
    for mut in ({3 + nnz - 7: "1 1 0.0"}, {3 + nnz // 2: lines[3 + 10]}, {3 + nnz + 250: "x"},
                {3 + nnz // 3: lines[3 + nnz // 4], 3 + nnz // 2: "bad"}):
        ls = list(lines)
        for i, t in mut.items():
            ls[i] = t
        t2 = "\n".join(ls) + "\n"
        assert _outcome(lambda s: binio.parse_problem(s, threads=16), t2) == _outcome(binio._parse_problem_py, t2)


def test_binary_roundtrip(tmp_path):
    p = generate(GenSpec(40, 80, 0.1, "socp4", seed=2))
    for canonical in (False, True):
        path = str(tmp_path / f"p{int(canonical)}.cfb")
        binio.write_problem_binary(path, p, canonical=canonical)
        for mm in (True, False):
            q = binio.read_problem_binary(path, mmap=mm)
            assert q.A.num_rows == 40 and q.A.num_cols == 80
            key = lambda a: np.lexsort((np.asarray(a.rows), np.asarray(a.cols)))  # noqa: E731
            for x, y in ((q.A.rows, p.A.rows), (q.A.cols, p.A.cols), (q.A.vals, p.A.vals)):
                assert np.array_equal(np.asarray(x)[key(q.A)], np.asarray(y)[key(p.A)])
            assert np.array_equal(q.b, p.b) and np.array_equal(q.c, p.c)
            assert tuple(q.cones.block_sizes) == tuple(p.cones.block_sizes)
    with open(path, "r+b") as f:
        f.write(b"NOTMAGIC")
    with pytest.raises(ValueError):
        binio.read_problem_binary(path)
    os.truncate(str(tmp_path / "p0.cfb"), 100)
    with pytest.raises(ValueError):
        binio.read_problem_binary(str(tmp_path / "p0.cfb"))


def test_native_path_covers_ascii_cases():
    """Only non-ASCII text and integers beyond int64 leave the native reader."""
    g = load_golden("coneprob_cases.npz")
    fallback = []
    for k, text in enumerate(g["texts"]):
        try:
            if binio._native(str(text), None) is None:
                fallback.append(k)
        except Exception:
            pass
    texts = [str(g["texts"][k]) for k in fallback]
    assert len(fallback) == 3
    assert all(any(ord(ch) > 127 for ch in t) or "99999999999999999999" in t for t in texts)


def test_write_solution_and_trace_csv_format():
    """write_solution (fileio.py:193-200) and trace_csv (:244-266): repr() per value."""
    from types import SimpleNamespace

    from paper_2203_05027_b200.binio import TRACE_COLUMNS, trace_csv, write_solution

    rng = np.random.default_rng(5)
    x = np.concatenate([rng.standard_normal(50) * 10.0 ** rng.integers(-30, 30, 50),
                        [0.0, -0.0, 1e16, 1.5e-7, 123456789.0, np.inf, -np.inf, np.nan]])
    lam = rng.standard_normal(7)
    got = write_solution("solved", 1.25, -0.1, 42, x, lam)
    want = "\n".join(["STATUS solved", "POBJ 1.25 / DOBJ -0.1 / ITERS 42"] +
                     [repr(float(v)) for v in x] + [repr(float(v)) for v in lam]) + "\n"
    assert got == want
    rep = SimpleNamespace(iter=25, status="running", **{c: 0.1 * k for k, c in enumerate(TRACE_COLUMNS[1:-1])})
    lines = trace_csv([rep, rep]).splitlines()
    assert lines[0] == ",".join(TRACE_COLUMNS)
    assert lines[1] == "25," + ",".join(repr(0.1 * k) for k in range(len(TRACE_COLUMNS) - 2)) + ",running"
