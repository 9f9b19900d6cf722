"""CPU checks of the parity checkers themselves (they must reject wrong kernels, not just pass right ones)."""
import numpy as np
import pytest

from oracle import objective as OO
from tests.helpers import assert_grad_rows, grad_rows_error


def test_grad_row_checker_has_teeth():
    g = np.random.default_rng(0)
    V, R = 131072, 3
    z = g.normal(0, 2.0, (R, V))
    toks = g.integers(0, V, R)
    coef = np.array([1e-3, -2e-4, 0.0])
    ref = OO.gradient_rows(z, None, toks, coef, [0.7] * R, z.shape)
    # an f32-rounded gradient passes at rtol 1e-5 ...
    assert assert_grad_rows(ref.astype(np.float32), z, toks, coef, [0.7] * R, 1e-5) < 1.0
    # ... a bf16-sized relative error on one tiny entry does not
    bad = ref.copy()
    j = int(np.argmin(np.abs(ref[0])))
    bad[0, j] *= 1.004
    assert grad_rows_error(bad, z, toks, coef, [0.7] * R, 1e-5)[0] > 1.0
    # a row whose slope is zero must be exactly zero
    bad = ref.copy()
    bad[2, 5] = 1e-20
    assert grad_rows_error(bad, z, toks, coef, [0.7] * R, 1e-5)[0] > 1.0
    # zeroing every non-target entry fails (the check inside assert_grad_rows)
    bad = np.zeros_like(ref)
    bad[np.arange(R), toks] = ref[np.arange(R), toks]
    with pytest.raises(AssertionError):
        assert_grad_rows(bad, z, toks, coef, [0.7] * R, 2.0 ** -8)
