"""Problem containers and validation — the input contract of the drop-in.

Same public types, fields, invariants and messages as the reference
``conefree.model`` (model.py:43-217), so a ``ProblemInstance`` built with
either package is accepted by either ``solve``:

* ``TripletMatrix`` (model.py:43-90): immutable COO with int64 rows/cols and
  float64 values, any entry order.
* ``ConeSpec`` (model.py:93-115): Lorentz block sizes; size 1 is R+.
  ``ConeSpec.orthant(n)`` keeps the sizes as a compact numpy array and only
  materialises the Python tuple when ``block_sizes`` is read, so a 10M-column
  LP does not pay for a 10M-element tuple on the solve path.
* ``ProblemInstance`` (model.py:118-137), ``ValidationReport`` (:140-149) and
  ``validate`` (:179-217), whose violation strings are reproduced verbatim
  because ``solve`` raises ``ValueError("invalid problem: " + first three)``
  (solver.py:300-302).

``validate`` here is the host restatement used for the *messages*; the solve
path runs the same checks on the GPU (cf_plan_create) and only calls this one
when the device reports a violation.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "TripletMatrix",
    "ConeSpec",
    "ProblemInstance",
    "ValidationReport",
    "validate",
    "triplet_violations",
    "cone_sizes_array",
]


def _readonly_1d(values, dtype) -> np.ndarray:
    arr = np.array(values, dtype=dtype)
    if arr.ndim != 1:
        raise ValueError(f"expected a 1-d array, got shape {arr.shape}")
    arr.setflags(write=False)
    return arr


@dataclass(frozen=True)
class TripletMatrix:
    """Sparse m-by-n matrix as parallel (row, col, value) arrays (zero-based)."""

    num_rows: int
    num_cols: int
    rows: np.ndarray
    cols: np.ndarray
    vals: np.ndarray

    def __post_init__(self):
        for name, dtype in (("rows", np.int64), ("cols", np.int64), ("vals", np.float64)):
            object.__setattr__(self, name, _readonly_1d(getattr(self, name), dtype))
        if len({self.rows.size, self.cols.size, self.vals.size}) != 1:
            raise ValueError("rows, cols, vals must have equal length")

    @property
    def nnz(self) -> int:
        return int(self.vals.size)

    @classmethod
    def _view(cls, num_rows, num_cols, rows, cols, vals):
        """Internal: wrap 1-d arrays of the right dtypes without the copy of __init__ (slices of
        a problem the caller already handed over, e.g. one rank's share in sharded.py)."""
        obj = object.__new__(cls)
        for name, v in (("num_rows", int(num_rows)), ("num_cols", int(num_cols)), ("rows", rows), ("cols", cols),
                        ("vals", vals)):
            object.__setattr__(obj, name, v)
        return obj

    @classmethod
    def from_entries(cls, num_rows, num_cols, entries):
        triples = list(entries)
        return cls(num_rows, num_cols, [t[0] for t in triples], [t[1] for t in triples],
                   [t[2] for t in triples])

    @classmethod
    def from_dense(cls, a):
        """Nonzeros of a dense array, enumerated column-major (canonical order)."""
        dense = np.asarray(a, dtype=np.float64)
        m, n = dense.shape
        cols, rows = np.nonzero(dense.T)
        return cls(m, n, rows, cols, dense[rows, cols])

    def to_dense(self):
        out = np.zeros((self.num_rows, self.num_cols))
        out[self.rows, self.cols] = self.vals
        return out


class ConeSpec:
    """Ordered Lorentz-cone block sizes partitioning the n variables."""

    __slots__ = ("_tuple", "_array")

    def __init__(self, block_sizes):
        if isinstance(block_sizes, np.ndarray):
            arr = np.asarray(block_sizes, dtype=np.int64).copy()
            arr.setflags(write=False)
            object.__setattr__(self, "_array", arr)
            object.__setattr__(self, "_tuple", None)
        else:
            object.__setattr__(self, "_tuple", tuple(int(s) for s in block_sizes))
            object.__setattr__(self, "_array", None)

    def __reduce__(self):   # picklable despite the immutable __setattr__ (process pools)
        return (ConeSpec, (self._array if self._array is not None else self._tuple,))

    @property
    def block_sizes(self) -> tuple:
        if self._tuple is None:
            object.__setattr__(self, "_tuple", tuple(self._array.tolist()))
        return self._tuple

    def sizes_array(self) -> np.ndarray:
        if self._array is None:
            arr = np.fromiter(self._tuple, dtype=np.int64, count=len(self._tuple))
            arr.setflags(write=False)
            object.__setattr__(self, "_array", arr)
        return self._array

    @property
    def dim(self) -> int:
        return int(self.sizes_array().sum())

    @classmethod
    def orthant(cls, n):
        """Nonnegative orthant R+^n: n blocks of size 1."""
        return cls(np.ones(int(n), dtype=np.int64))

    def __eq__(self, other):
        if not hasattr(other, "block_sizes"):
            return NotImplemented
        return np.array_equal(self.sizes_array(), cone_sizes_array(other))

    def __hash__(self):
        return hash(self.sizes_array().tobytes())

    def __repr__(self):
        arr = self.sizes_array()
        if arr.size > 8:
            return f"ConeSpec(<{arr.size} blocks, dim {int(arr.sum())}>)"
        return f"ConeSpec(block_sizes={self.block_sizes})"

    def __setattr__(self, name, value):
        raise AttributeError("ConeSpec is immutable")


def cone_sizes_array(cones) -> np.ndarray:
    """int64 block sizes of this package's ConeSpec or any object with ``block_sizes``."""
    if isinstance(cones, ConeSpec):
        return cones.sizes_array()
    sizes = cones.block_sizes
    return np.fromiter((int(s) for s in sizes), dtype=np.int64, count=len(sizes))


@dataclass(frozen=True)
class ProblemInstance:
    """minimize c.x  subject to  A x = b,  x in K (model.py:3-11)."""

    A: TripletMatrix
    b: np.ndarray
    c: np.ndarray
    cones: ConeSpec

    def __post_init__(self):
        object.__setattr__(self, "b", _readonly_1d(self.b, np.float64))
        object.__setattr__(self, "c", _readonly_1d(self.c, np.float64))

    @classmethod
    def _view(cls, A, b, c, cones):
        """Internal: no copies (see TripletMatrix._view)."""
        obj = object.__new__(cls)
        for name, v in (("A", A), ("b", b), ("c", c), ("cones", cones)):
            object.__setattr__(obj, name, v)
        return obj

    @property
    def m(self) -> int:
        return self.A.num_rows

    @property
    def n(self) -> int:
        return self.A.num_cols


@dataclass(frozen=True)
class ValidationReport:
    """Violations are errors, warnings are not (model.py:140-149)."""

    violations: tuple = ()
    warnings: tuple = ()

    @property
    def ok(self) -> bool:
        return len(self.violations) == 0


def triplet_violations(a) -> list:
    """Index/finiteness/zero/duplicate checks of model.py:152-176, same order and text."""
    m, n, o = a.num_rows, a.num_cols, int(a.vals.size)
    rows, cols, vals = a.rows, a.cols, a.vals
    msgs = []
    msgs += [f"entry {k}: row index {rows[k]} outside [0, {m})"
             for k in np.flatnonzero((rows < 0) | (rows >= m))]
    msgs += [f"entry {k}: column index {cols[k]} outside [0, {n})"
             for k in np.flatnonzero((cols < 0) | (cols >= n))]
    msgs += [f"entry {k}: value {vals[k]} is not finite" for k in np.flatnonzero(~np.isfinite(vals))]
    msgs += [f"entry {k}: zero value at ({rows[k]}, {cols[k]})" for k in np.flatnonzero(vals == 0.0)]
    if o:
        key = rows * np.int64(max(n, 1)) + cols
        _, first = np.unique(key, return_index=True)
        if first.size != o:
            is_first = np.zeros(o, dtype=bool)
            is_first[first] = True
            msgs += [f"duplicate entry at ({rows[k]}, {cols[k]})" for k in np.flatnonzero(~is_first)]
    return msgs


def validate(p) -> ValidationReport:
    """Every invariant of a problem instance; returns data, never raises (model.py:179-217)."""
    a = p.A
    m, n = a.num_rows, a.num_cols
    violations = triplet_violations(a)
    if p.b.size != m:
        violations.append(f"b has length {p.b.size} != m={m}")
    if p.c.size != n:
        violations.append(f"c has length {p.c.size} != n={n}")
    for name, vec in (("b", p.b), ("c", p.c)):
        violations += [f"{name}[{k}] = {vec[k]} is not finite" for k in np.flatnonzero(~np.isfinite(vec))]
    sizes = cone_sizes_array(p.cones)
    violations += [f"cone block {i} has size {s} < 1" for i, s in zip(np.flatnonzero(sizes < 1), sizes[sizes < 1])]
    total = int(sizes.sum())
    if total != n:
        violations.append(f"cone sizes sum {total} != n={n}")
    warnings = []
    if m > 0:
        inside = (a.rows >= 0) & (a.rows < m)
        per_row = np.bincount(a.rows[inside], minlength=m)
        warnings = [f"row {i} of A has no nonzeros" for i in np.flatnonzero(per_row == 0)]
    return ValidationReport(tuple(violations), tuple(warnings))
