"""TEST INFRASTRUCTURE ONLY — CPU oracle for the parity tests.

A numpy restatement of the reference solver's hot path (``conefree``,
arXiv 2203.05027) in its literal per-nonzero form: the o-length y and gamma
vectors are stored and updated exactly as solver.py:168-197 does. It is
PINNED against fixtures produced by running the unmodified reference
(tests/golden/*.npz, made by tests/golden/make_golden.py) — see
tests/test_oracle_golden.py.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (``cpu_baseline`` / ``--impl reference``) may import this package, and
only as the checker or the timed CPU baseline. The product path
(``paper_2203_05027_b200``) never imports it.
"""

from .port import (  # noqa: F401
    Factors,
    OracleState,
    apply_U,
    apply_Ut,
    apply_V,
    apply_Vt,
    apply_y_factor,
    build_factors,
    check_termination,
    compute_report,
    dense_iterate,
    iterate,
    project_block,
    project_product,
    solve,
    step,
)
