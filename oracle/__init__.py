"""CPU oracle for the rolloutlab hot path -- TEST INFRASTRUCTURE ONLY.

A numpy/float64 restatement of the reference algorithm (pkg/src/rolloutlab/{core,fusion,objective,
toy_env}.py), each function citing the reference lines it follows.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU-baseline / `--impl reference` arm may import it, and
only as the checker or the timed CPU reference -- never as part of the product path (the package
`paper_2509_18883_b200` does not import it and has no CPU fallback).

Pinning: the restatement is checked against golden vectors generated from the unmodified reference
(tests/golden/make_golden.py -> tests/golden/*.npz|json) in tests/test_oracle_golden.py.
Set OPENBLAS_NUM_THREADS=1: the reference's own norms (np.linalg.norm -> OpenBLAS ddot) change in the
last ulp with the BLAS thread count.
"""

import os as _os

_os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
try:  # numpy may already be loaded with a multi-threaded BLAS: pin it at runtime as well
    from threadpoolctl import threadpool_limits as _tpl

    _BLAS_LIMIT = _tpl(limits=1, user_api="blas")
except Exception:  # pragma: no cover
    _BLAS_LIMIT = None
