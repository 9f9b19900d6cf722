"""Drop-in fidelity: SPEC.md's worked examples, written against `rolloutlab`'s API
(tests/dropin_examples.py), run unchanged through an import swap onto this package -- checked against
the values SPEC.md states and, where the unmodified reference is importable (baseline/_ref, the
install that travels with the repo), against the reference's own results on the same calls."""
import sys
from pathlib import Path

import numpy as np
import pytest

from tests import dropin_examples as D

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _reference_results():
    for cand in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (cand / "rolloutlab").exists():
            sys.path.insert(0, str(cand))
            try:
                for k in [k for k in sys.modules if k == "rolloutlab" or k.startswith("rolloutlab.")]:
                    del sys.modules[k]
                return D.run_examples()
            finally:
                sys.path.remove(str(cand))
                for k in [k for k in sys.modules if k == "rolloutlab" or k.startswith("rolloutlab.")]:
                    del sys.modules[k]
    return None


def test_spec_examples_through_import_swap(cuda):
    with D.swap_in():
        ours = D.run_examples()
    for k, want in D.SPEC_EXPECTED.items():
        np.testing.assert_allclose(np.asarray(ours[k], dtype=np.float64).reshape(np.shape(want)), want,
                                   rtol=1e-12, atol=1e-15, err_msg=k)
    # the surviving p = 0.5 entries are rescaled 0.4 -> 0.8 (SPEC dropout example)
    kept = ours["dropout/p05"][ours["dropout/p05"] != 0]
    assert kept.size and np.allclose(kept, 0.8, rtol=1e-15)
    ref = _reference_results()
    if ref is None:
        pytest.skip("unmodified reference not importable here; SPEC values checked")
    assert set(ref) == set(ours)
    for k in ref:
        a, b = np.asarray(ours[k], dtype=np.float64), np.asarray(ref[k], dtype=np.float64)
        assert a.shape == b.shape, k
        if k.startswith(("dropout/", "erase/", "fuse/kept", "fuse/erased", "adv/", "obj/advantages", "tis/", "clip/")):
            assert np.array_equal(a, b), k  # integer / exact decisions
        else:
            np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-15, err_msg=k)
