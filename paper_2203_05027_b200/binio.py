"""Problem file I/O: the reference's CONEPROB text format, natively, plus a binary format.

Text (``conefree/fileio.py:1-25``):

* ``parse_problem(text)`` / ``read_problem(path)`` are the reference's
  ``parse_problem`` (fileio.py:98-190). They raise the same ``ParseError(line,
  message)`` for the same first bad line, with the same message. The work is done
  by the multi-threaded C++ reader in ``csrc/cf_io.cpp`` (``cf_coneprob_*`` in
  include/cfb200.h). Inputs outside its subset (non-ASCII text, integers beyond
  int64) go through ``_parse_problem_py``, a line-by-line restatement of
  fileio.py:98-190.
* ``write_problem(p)`` / ``write_problem_file(path, p)`` restate
  write_problem (fileio.py:56-72): canonical entry order and Python ``repr``
  floats, so write -> parse reproduces every value bit for bit.

Binary (beside CONEPROB): ``write_problem_binary`` /
``read_problem_binary``. Layout, little-endian:

* magic ``b"CFPROB\\x00\\x01"``;
* int64 header ``m, n, nnz, n_blocks, flags``, with flags bit 0 set when the
  entries are in canonical order;
* the arrays at 64-byte-aligned offsets: rows i64[nnz], cols i64[nnz],
  vals f64[nnz], b f64[m], c f64[n], block_sizes i64[n_blocks].

``read_problem_binary(path, mmap=True)`` maps the arrays without copying. The
problem is validated (``validate``, model.py:179-217) unless ``validate=False``.
"""

from __future__ import annotations

import ctypes
import os
import tempfile

import numpy as np

from .problem import ConeSpec, ProblemInstance, TripletMatrix, validate

__all__ = [
    "ParseError",
    "parse_problem",
    "read_problem",
    "write_problem",
    "write_problem_file",
    "format_float",
    "write_problem_binary",
    "read_problem_binary",
    "write_solution",
    "write_solution_file",
    "TRACE_COLUMNS",
    "trace_csv",
]

CF_IO_PARSE = 6
CF_IO_FALLBACK = 7
MAGIC = b"CFPROB\x00\x01"
_ALIGN = 64


class ParseError(ValueError):
    """Malformed file; carries the 1-based offending line number (fileio.py:43-49)."""

    def __init__(self, line: int, message: str):
        self.line = line
        self.message = message
        super().__init__(f"line {line}: {message}")


# ---------------------------------------------------------------- native reader
def _native(text: str | None, path: str | None, threads: int = 0) -> ProblemInstance | None:
    """The C++ reader; None when the input needs the Python restatement."""
    from ._lib import lib

    L = lib()
    handle = ctypes.c_void_p()
    if path is not None:
        rc = L.cf_coneprob_open(os.fsencode(path), None, 0, ctypes.byref(handle))
        if rc:
            raise OSError(f"cannot open {path!r}")
    else:
        raw = text.encode("utf-8", "surrogatepass")
        rc = L.cf_coneprob_open(None, raw, len(raw), ctypes.byref(handle))
        if rc:
            raise MemoryError("cf_coneprob_open failed")
    try:
        dims = (ctypes.c_int64 * 4)()
        line = ctypes.c_int64(0)
        msg = ctypes.create_string_buffer(4096)
        rc = L.cf_coneprob_header(handle, dims, ctypes.byref(line), msg, len(msg))
        if rc == CF_IO_FALLBACK:
            return None
        if rc == CF_IO_PARSE:
            raise ParseError(int(line.value), msg.value.decode("utf-8", "replace"))
        if rc:
            raise RuntimeError(f"cf_coneprob_header failed ({rc})")
        m, n, nnz, nb = (int(v) for v in dims)
        sizes = np.empty(nb, dtype=np.int64)
        L.cf_coneprob_sizes(handle, ctypes.c_void_p(sizes.ctypes.data))
        rows = np.empty(nnz, dtype=np.int64)
        cols = np.empty(nnz, dtype=np.int64)
        vals = np.empty(nnz, dtype=np.float64)
        b = np.empty(m, dtype=np.float64)
        c = np.empty(n, dtype=np.float64)

        def ptr(a):
            return ctypes.c_void_p(a.ctypes.data)

        rc = L.cf_coneprob_body(handle, ptr(rows), ptr(cols), ptr(vals), ptr(b), ptr(c), int(threads),
                                ctypes.byref(line), msg, len(msg))
        if rc == CF_IO_FALLBACK:
            return None
        if rc == CF_IO_PARSE:
            raise ParseError(int(line.value), msg.value.decode("utf-8", "replace"))
        if rc:
            raise RuntimeError(f"cf_coneprob_body failed ({rc})")
    finally:
        L.cf_coneprob_close(handle)
    # every validate() invariant was checked line by line above (bounds, finite,
    # nonzero, duplicates, vector lengths, cone sizes), so validate cannot fail here
    return ProblemInstance(A=TripletMatrix(m, n, rows, cols, vals), b=b, c=c, cones=ConeSpec(sizes))


def parse_problem(text: str, threads: int = 0) -> ProblemInstance:
    """Parse a CONEPROB text (fileio.py:98-190), reporting the offending line on error."""
    p = _native(text, None, threads)
    return p if p is not None else _parse_problem_py(text)


def read_problem(path: str, threads: int = 0) -> ProblemInstance:
    """Parse a CONEPROB file, memory-mapped (same errors as parse_problem)."""
    p = _native(None, path, threads)
    if p is not None:
        return p
    with open(path, encoding="utf-8") as f:
        return _parse_problem_py(f.read())


# ---------------------------------------------------------------- Python restatement (fallback)
def _content_lines(text):
    for num, raw in enumerate(text.splitlines(), start=1):
        stripped = raw.strip()
        if stripped and not stripped.startswith("#"):
            yield num, stripped


def _int(tok, line, what):
    try:
        return int(tok)
    except ValueError:
        raise ParseError(line, f"expected integer {what}, got {tok!r}") from None


def _float(tok, line, what):
    try:
        return float(tok)
    except ValueError:
        raise ParseError(line, f"expected number {what}, got {tok!r}") from None


def _parse_problem_py(text: str) -> ProblemInstance:
    """Line-by-line restatement of fileio.parse_problem (fileio.py:98-190)."""
    lines = _content_lines(text)

    def take(what):
        for item in lines:
            return item
        raise ParseError(0, f"file ended before {what}")

    num, header = take("header")
    if header != "CONEPROB 1":
        raise ParseError(num, f"expected 'CONEPROB 1' header, got {header!r}")
    num, dims = take("dimensions")
    toks = dims.split()
    if len(toks) != 3:
        raise ParseError(num, f"expected 'm n nnz', got {dims!r}")
    m, n, nnz = _int(toks[0], num, "m"), _int(toks[1], num, "n"), _int(toks[2], num, "nnz")
    if m < 1 or n < 1 or nnz < 0:
        raise ParseError(num, f"bad dimensions m={m} n={n} nnz={nnz}")
    num, cone_line = take("CONES line")
    toks = cone_line.split()
    if not toks or toks[0] != "CONES":
        raise ParseError(num, f"expected 'CONES ...', got {cone_line!r}")
    if len(toks) < 2:
        raise ParseError(num, "CONES line missing block count")
    count = _int(toks[1], num, "cone block count")
    if len(toks) != 2 + count:
        raise ParseError(num, f"CONES declares {count} blocks but lists {len(toks) - 2}")
    sizes = [_int(t, num, "cone size") for t in toks[2:]]
    for s in sizes:
        if s < 1:
            raise ParseError(num, f"cone size {s} < 1")
    if sum(sizes) != n:
        raise ParseError(num, f"cone sizes sum {sum(sizes)} != n={n}")
    rows = np.empty(nnz, dtype=np.int64)
    cols = np.empty(nnz, dtype=np.int64)
    vals = np.empty(nnz, dtype=np.float64)
    seen = set()
    for k in range(nnz):
        num, entry = take(f"entry {k}")
        toks = entry.split()
        if len(toks) != 3:
            raise ParseError(num, f"expected 'i j value', got {entry!r}")
        i = _int(toks[0], num, "row index")
        j = _int(toks[1], num, "column index")
        v = _float(toks[2], num, "value")
        if not 0 <= i < m:
            raise ParseError(num, f"row index {i} outside [0, {m})")
        if not 0 <= j < n:
            raise ParseError(num, f"column index {j} outside [0, {n})")
        if not np.isfinite(v):
            raise ParseError(num, f"value {toks[2]} is not finite")
        if v == 0.0:
            raise ParseError(num, f"zero value at ({i}, {j})")
        if (i, j) in seen:
            raise ParseError(num, f"duplicate entry at ({i}, {j})")
        seen.add((i, j))
        rows[k], cols[k], vals[k] = i, j, v

    def vector(length, name):
        out = np.empty(length)
        for idx in range(length):
            num, tok = take(f"{name}[{idx}]")
            v = _float(tok, num, f"{name}[{idx}]")
            if not np.isfinite(v):
                raise ParseError(num, f"{name}[{idx}] = {tok} is not finite")
            out[idx] = v
        return out

    b = vector(m, "b")
    c = vector(n, "c")
    for num, extra in lines:
        raise ParseError(num, f"unexpected trailing content {extra!r}")
    p = ProblemInstance(A=TripletMatrix(m, n, rows, cols, vals), b=b, c=c, cones=ConeSpec(tuple(sizes)))
    rep = validate(p)
    if not rep.ok:
        raise ParseError(0, "; ".join(rep.violations[:3]))
    return p


# ---------------------------------------------------------------- writer
def format_float(v: float) -> str:
    """repr(float(v)) through the native formatter (fileio.py:52-53)."""
    from ._lib import lib

    buf = ctypes.create_string_buffer(64)
    n = lib().cf_format_double(float(v), buf)
    return buf.raw[:n].decode("ascii")


def _canonical(p):
    a = p.A
    rows = np.asarray(a.rows, dtype=np.int64)
    cols = np.asarray(a.cols, dtype=np.int64)
    vals = np.asarray(a.vals, dtype=np.float64)
    order = np.lexsort((rows, cols))   # fileio.py:59
    return (np.ascontiguousarray(rows[order]), np.ascontiguousarray(cols[order]),
            np.ascontiguousarray(vals[order]))


def write_problem_file(path: str, p, threads: int = 0) -> None:
    """Serialize an instance to `path` (write_problem, fileio.py:56-72), all host cores."""
    from ._lib import lib

    rows, cols, vals = _canonical(p)
    b = np.ascontiguousarray(p.b, dtype=np.float64)
    c = np.ascontiguousarray(p.c, dtype=np.float64)
    sizes = np.ascontiguousarray(np.asarray(p.cones.block_sizes, dtype=np.int64))

    def ptr(a):
        return ctypes.c_void_p(a.ctypes.data) if a.size else ctypes.c_void_p(0)

    rc = lib().cf_coneprob_write(os.fsencode(path), int(p.A.num_rows), int(p.A.num_cols), int(rows.size),
                                 ptr(rows), ptr(cols), ptr(vals), ptr(b), ptr(c), int(sizes.size), ptr(sizes),
                                 int(threads))
    if rc:
        raise OSError(f"cannot write {path!r}")


def write_problem(p, threads: int = 0) -> str:
    """The CONEPROB text of an instance (fileio.py:56-72)."""
    fd, path = tempfile.mkstemp(prefix="coneprob_", suffix=".txt")
    os.close(fd)
    try:
        write_problem_file(path, p, threads)
        with open(path, encoding="ascii") as f:
            return f.read()
    finally:
        os.unlink(path)


def _solution_head(status: str, pobj: float, dobj: float, iters: int) -> str:
    return f"STATUS {status}\nPOBJ {repr(float(pobj))} / DOBJ {repr(float(dobj))} / ITERS {iters}\n"


def write_solution_file(path: str, status: str, pobj: float, dobj: float, iters: int, x, lam,
                        threads: int = 0) -> None:
    """write_solution (fileio.py:193-200) straight to `path`; the x and lam lines are
    formatted by the native writer on all host cores."""
    from ._lib import lib

    x = np.ascontiguousarray(x, dtype=np.float64)
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    head = _solution_head(status, pobj, dobj, iters).encode("utf-8")
    rc = lib().cf_solution_write(os.fsencode(path), head,
                                 ctypes.c_void_p(x.ctypes.data) if x.size else ctypes.c_void_p(0), int(x.size),
                                 ctypes.c_void_p(lam.ctypes.data) if lam.size else ctypes.c_void_p(0), int(lam.size),
                                 int(threads))
    if rc:
        raise OSError(f"cannot write {path!r}")


def write_solution(status: str, pobj: float, dobj: float, iters: int, x, lam) -> str:
    """The solution text (fileio.py:193-200): STATUS, POBJ/DOBJ/ITERS, x, lam."""
    fd, path = tempfile.mkstemp(prefix="conesol_", suffix=".txt")
    os.close(fd)
    try:
        write_solution_file(path, status, pobj, dobj, iters, x, lam)
        with open(path, encoding="utf-8") as f:
            return f.read()
    finally:
        os.unlink(path)


TRACE_COLUMNS = (
    "iter",
    "prim_res_inf",
    "prim_res_2",
    "dual_res_inf",
    "dual_res_2",
    "stat_res_inf",
    "stat_res_2",
    "cone_gap",
    "pobj",
    "dobj",
    "gap",
    "status",
)


def trace_csv(trace) -> str:
    """Per-report CSV of a solve's trace (fileio.py:228-266), no timing columns."""
    lines = [",".join(TRACE_COLUMNS)]
    for rep in trace:
        cells = [str(rep.iter)]
        cells.extend(repr(float(getattr(rep, col))) for col in TRACE_COLUMNS[1:-1])
        cells.append(rep.status)
        lines.append(",".join(cells))
    return "\n".join(lines) + "\n"


# ---------------------------------------------------------------- binary format
def _pad(off: int) -> int:
    return -(-off // _ALIGN) * _ALIGN


def write_problem_binary(path: str, p, canonical: bool = False) -> None:
    """Write the binary problem file (layout in the module docstring)."""
    a = p.A
    if canonical:
        rows, cols, vals = _canonical(p)
    else:
        rows = np.asarray(a.rows, dtype=np.int64)
        cols = np.asarray(a.cols, dtype=np.int64)
        vals = np.asarray(a.vals, dtype=np.float64)
    sizes = np.asarray(p.cones.block_sizes, dtype=np.int64)
    arrays = [rows.astype("<i8", copy=False), cols.astype("<i8", copy=False), vals.astype("<f8", copy=False),
              np.asarray(p.b, dtype="<f8"), np.asarray(p.c, dtype="<f8"), sizes.astype("<i8", copy=False)]
    head = np.array([a.num_rows, a.num_cols, rows.size, sizes.size, 1 if canonical else 0], dtype="<i8")
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(head.tobytes())
        off = len(MAGIC) + head.nbytes
        for arr in arrays:
            start = _pad(off)
            f.write(b"\0" * (start - off))
            f.write(np.ascontiguousarray(arr).tobytes())
            off = start + arr.nbytes


def read_problem_binary(path: str, mmap: bool = True, validate_problem: bool = True) -> ProblemInstance:
    """Read a binary problem file; the arrays are memory-mapped unless mmap=False."""
    with open(path, "rb") as f:
        magic = f.read(len(MAGIC))
        if magic != MAGIC:
            raise ValueError(f"{path!r} is not a binary problem file (magic {magic!r})")
        head = np.frombuffer(f.read(5 * 8), dtype="<i8")
    if head.size != 5:
        raise ValueError(f"{path!r}: truncated header")
    m, n, nnz, nb, _flags = (int(v) for v in head)
    if m < 0 or n < 0 or nnz < 0 or nb < 0:
        raise ValueError(f"{path!r}: bad header {head.tolist()}")
    specs = [("<i8", nnz), ("<i8", nnz), ("<f8", nnz), ("<f8", m), ("<f8", n), ("<i8", nb)]
    off = len(MAGIC) + 5 * 8
    need = off
    for dt, cnt in specs:
        need = _pad(need) + 8 * cnt
    if os.path.getsize(path) < need:
        raise ValueError(f"{path!r}: truncated ({os.path.getsize(path)} < {need} bytes)")
    out = []
    for dt, cnt in specs:
        start = _pad(off)
        if mmap and cnt:
            out.append(np.memmap(path, dtype=dt, mode="r", offset=start, shape=(cnt,)))
        else:
            out.append(np.fromfile(path, dtype=dt, count=cnt, offset=start))
        off = start + 8 * cnt
    rows, cols, vals, b, c, sizes = out
    p = ProblemInstance(A=TripletMatrix(m, n, rows, cols, vals), b=b, c=c, cones=ConeSpec(np.asarray(sizes)))
    if validate_problem:
        rep = validate(p)
        if not rep.ok:
            raise ValueError("invalid problem: " + "; ".join(rep.violations[:3]))
    return p
