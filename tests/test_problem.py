"""Host-side input contract (CPU): mirrors the reference's own tests pkg/tests/test_model.py
against this package's types, plus duck-typing of the reference's container shapes."""

import numpy as np
import pytest

from paper_2203_05027_b200 import ConeSpec, ProblemInstance, TripletMatrix, validate

DEMO = np.array([[1.0, 0.0, 4.0, 6.0, 8.0], [0.0, 0.0, 5.0, 0.0, 0.0], [2.0, 3.0, 0.0, 7.0, 0.0]])


def demo_problem(cones=None, b=None, c=None, a=None):
    a = a or TripletMatrix.from_dense(DEMO)
    return ProblemInstance(A=a, b=np.zeros(3) if b is None else b, c=np.zeros(5) if c is None else c,
                           cones=cones or ConeSpec.orthant(5))


def test_validate_ok_example1():
    rep = validate(demo_problem())
    assert rep.ok and rep.violations == () and rep.warnings == ()


def test_cone_sum_mismatch():
    rep = validate(demo_problem(cones=ConeSpec((4,))))
    assert rep.violations == ("cone sizes sum 4 != n=5",)


def test_duplicates_reported():
    a = TripletMatrix(2, 2, [0, 1, 0], [0, 1, 0], [1.0, 2.0, 3.0])
    rep = validate(ProblemInstance(a, np.zeros(2), np.zeros(2), ConeSpec.orthant(2)))
    assert rep.violations == ("duplicate entry at (0, 0)",)


def test_out_of_range_indices():
    a = TripletMatrix(2, 2, [0, 2, -1], [0, 1, 5], [1.0, 2.0, 3.0])
    rep = validate(ProblemInstance(a, np.zeros(2), np.zeros(2), ConeSpec.orthant(2)))
    assert rep.violations[:3] == ("entry 1: row index 2 outside [0, 2)", "entry 2: row index -1 outside [0, 2)",
                                  "entry 2: column index 5 outside [0, 2)")


def test_zero_and_nonfinite_values():
    a = TripletMatrix(2, 2, [0, 1, 1], [0, 0, 1], [0.0, np.inf, np.nan])
    rep = validate(ProblemInstance(a, np.zeros(2), np.zeros(2), ConeSpec.orthant(2)))
    assert rep.violations == ("entry 1: value inf is not finite", "entry 2: value nan is not finite",
                              "entry 0: zero value at (0, 0)")


def test_vector_lengths_and_finiteness():
    rep = validate(demo_problem(b=np.zeros(2), c=np.array([0, 0, 0, 0, np.nan])))
    assert "b has length 2 != m=3" in rep.violations
    assert "c[4] = nan is not finite" in rep.violations


def test_empty_row_is_warning():
    a = TripletMatrix(3, 2, [0, 2], [0, 1], [1.0, 1.0])
    rep = validate(ProblemInstance(a, np.zeros(3), np.zeros(2), ConeSpec.orthant(2)))
    assert rep.ok and rep.warnings == ("row 1 of A has no nonzeros",)


def test_block_size_below_one():
    rep = validate(demo_problem(cones=ConeSpec((0, 5))))
    assert rep.violations == ("cone block 0 has size 0 < 1",)


def test_validate_is_pure():
    p = demo_problem()
    assert validate(p) == validate(p)


def test_containers_are_immutable():
    a = TripletMatrix.from_dense(DEMO)
    with pytest.raises(ValueError):
        a.vals[0] = 5.0
    with pytest.raises(Exception):
        a.num_rows = 4
    with pytest.raises(AttributeError):
        ConeSpec((1, 2))._tuple = (3,)
    p = demo_problem()
    with pytest.raises(ValueError):
        p.b[0] = 1.0


def test_from_dense_round_trip_canonical_order():
    a = TripletMatrix.from_dense(DEMO)
    np.testing.assert_array_equal(a.to_dense(), DEMO)
    np.testing.assert_array_equal(a.vals, np.arange(1.0, 9.0))  # column-major enumeration


def test_mismatched_lengths():
    with pytest.raises(ValueError, match="equal length"):
        TripletMatrix(2, 2, [0, 1], [0], [1.0, 2.0])
    with pytest.raises(ValueError, match="1-d"):
        TripletMatrix(2, 2, [[0, 1]], [[0, 1]], [[1.0, 2.0]])


def test_conespec_compact_orthant_matches_tuple():
    big = ConeSpec.orthant(1000)
    assert big == ConeSpec((1,) * 1000)
    assert big.block_sizes == (1,) * 1000 and big.dim == 1000
    assert ConeSpec((4, 4)).sizes_array().tolist() == [4, 4]


def test_problem_types_pickle():
    """Problems travel to process pools (the reference's run_bench scheme)."""
    import pickle

    from paper_2203_05027_b200 import ConeSpec, GenSpec, generate

    p = generate(GenSpec(20, 40, 0.1, "socp4", seed=1))
    q = pickle.loads(pickle.dumps(p))
    assert q.cones.block_sizes == p.cones.block_sizes and q.A.nnz == p.A.nnz
    assert (q.A.vals == p.A.vals).all() and (q.b == p.b).all()
    assert pickle.loads(pickle.dumps(ConeSpec((1, 2, 3)))).block_sizes == (1, 2, 3)
