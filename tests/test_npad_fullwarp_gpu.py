"""The one-warp full-diagonal driver (npad_fullwarp.cu, n <= 64: BASELINE
config 1) against the oracle and against the single-CTA rows driver, bit for
bit (pivots, matrix, unitary)."""
import os

import numpy as np
import pytest

from conftest import rel_fro
from oracle import npad_oracle

pytestmark = pytest.mark.gpu
TOL_F = 1e-10


@pytest.fixture(scope="module")
def E():
    import paper_2411_09982_b200 as eff

    return eff


@pytest.fixture
def driver():
    def _set(val):
        if val is None:
            os.environ.pop("QCH_NPAD_DRIVER", None)
        else:
            os.environ["QCH_NPAD_DRIVER"] = val

    old = os.environ.get("QCH_NPAD_DRIVER")
    yield _set
    _set(old)


def _herm(n, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    h = (a + a.conj().T) * (0.5 * scale)
    h = np.triu(h) + np.triu(h, 1).conj().T  # bitwise Hermitian
    return h + np.diag(np.arange(n, dtype=float))


def test_config1_vs_oracle(E, driver):
    driver(None)
    h = E.transmon_resonator_hamiltonian(3, 20).data
    ref = npad_oracle.run_incremental(h, tol=1e-12)
    st, piv = E.npad_run_logged(E.HermitianOperator(h), tol=1e-12, pivot_cap=ref["applied"])
    assert st.applied == ref["applied"] and st.converged
    np.testing.assert_array_equal(piv, ref["pivots"])
    assert rel_fro(st.current.data, ref["h"]) <= TOL_F


@pytest.mark.parametrize("n", [1, 2, 5, 31, 32, 33, 60, 64])
def test_random_vs_block_driver_bitwise(E, driver, n):
    h = _herm(n, 100 + n)
    driver(None)
    a, pa = E.npad_run_logged(E.HermitianOperator(h), tol=1e-12, track_unitary=True)
    driver("block")
    b, pb = E.npad_run_logged(E.HermitianOperator(h), tol=1e-12, track_unitary=True)
    assert a.applied == b.applied and a.converged == b.converged
    np.testing.assert_array_equal(pa, pb)
    np.testing.assert_array_equal(a.current.data, b.current.data)
    np.testing.assert_array_equal(a.accumulated_unitary, b.accumulated_unitary)


@pytest.mark.parametrize("n,iters", [(48, 300), (64, 5000)])
def test_random_vs_oracle(E, driver, n, iters):
    driver(None)
    h = _herm(n, n)
    ref = npad_oracle.run_incremental(h, tol=1e-12, max_iter=iters)
    st, piv = E.npad_run_logged(E.HermitianOperator(h), tol=1e-12, max_iter=iters)
    np.testing.assert_array_equal(piv, ref["pivots"])
    assert st.applied == ref["applied"] and st.converged == ref["converged"]
    assert rel_fro(st.current.data, ref["h"]) <= TOL_F


def test_ties_and_zero_rows(E, driver):
    # exact magnitude ties (equal couplings) and rows with no coupling at all
    n = 40
    h = np.diag(np.arange(n, dtype=float)).astype(complex)
    for k in range(0, n - 1, 3):
        h[k + 1, k] = 0.25 * (1 + 1j) / np.sqrt(2)
        h[k, k + 1] = np.conj(h[k + 1, k])
    ref = npad_oracle.run_incremental(h, tol=1e-12)
    driver(None)
    st, piv = E.npad_run_logged(E.HermitianOperator(h), tol=1e-12, pivot_cap=max(ref["applied"], 1))
    np.testing.assert_array_equal(piv[: ref["applied"]], ref["pivots"])
    assert rel_fro(st.current.data, ref["h"]) <= TOL_F


def test_batch_one_warp_per_chain(E, driver):
    driver(None)
    mats = [_herm(50, 7 + k) for k in range(6)]
    res = E.npad_run_batch([E.HermitianOperator(m) for m in mats], tol=1e-12)
    for k, m in enumerate(mats):
        ref = npad_oracle.run_incremental(m, tol=1e-12)
        assert res.applied[k] == ref["applied"] and res.converged[k]
        assert rel_fro(res.operator(k).data, ref["h"]) <= TOL_F
