"""The whole-GPU single-chain driver (npad_coop.cu: one CTA per SM, one grid
barrier per rotation) — BASELINE config 3 — against the oracle and against
the single-CTA driver, bit for bit."""
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
def coop_env():
    def _set(val):
        if val is None:
            os.environ.pop("QCH_NPAD_COOP", None)
        else:
            os.environ["QCH_NPAD_COOP"] = val

    old = os.environ.get("QCH_NPAD_COOP")
    yield _set
    _set(old)


def _herm(n, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    h = (a + a.conj().T) * 0.05
    h = np.triu(h) + np.triu(h, 1).conj().T  # bitwise Hermitian
    return h + np.diag(np.linspace(0.0, 10.0, n))


def test_config3_prefix_vs_oracle(E, coop_env):
    # BASELINE config 3 operator (transmon 4 x resonator 1024, dim 4096), the
    # first 2000 greedy rotations
    coop_env("1")
    h = E.transmon_resonator_hamiltonian(4, 1024).data
    ref = npad_oracle.run_incremental(h, tol=1e-12, max_iter=2000)
    st, piv = E.npad_run_logged(E.HermitianOperator(h, validate=False), tol=1e-12, max_iter=2000)
    assert st.applied == 2000 and not st.converged
    np.testing.assert_array_equal(piv, ref["pivots"])
    assert rel_fro(st.current.data, ref["h"]) <= TOL_F


def test_dim1024_full_solve_vs_oracle(E, coop_env):
    coop_env("1")
    h = E.transmon_resonator_hamiltonian(4, 256).data
    ref = npad_oracle.run_incremental(h, tol=1e-12)
    st, piv = E.npad_run_logged(E.HermitianOperator(h), tol=1e-12, pivot_cap=ref["applied"])
    assert st.applied == ref["applied"] and st.converged
    np.testing.assert_array_equal(piv, ref["pivots"])
    assert rel_fro(st.current.data, ref["h"]) <= TOL_F
    ev_ref = np.sort(np.linalg.eigvalsh(h))
    assert np.max(np.abs(np.sort(st.current.diagonal()) - ev_ref)) <= 1e-10 * np.max(np.abs(ev_ref))


@pytest.mark.parametrize("n,iters", [(1100, 3000), (157, 4000)])
def test_random_vs_oracle(E, coop_env, n, iters):
    coop_env("1")
    h = _herm(n, n)
    ref = npad_oracle.run_incremental(h, tol=1e-12, max_iter=iters)
    st, piv = E.npad_run_logged(E.HermitianOperator(h), tol=1e-12, max_iter=iters)
    np.testing.assert_array_equal(piv, ref["pivots"])
    assert st.applied == ref["applied"] and st.converged == ref["converged"]
    assert rel_fro(st.current.data, ref["h"]) <= TOL_F


def test_coop_bit_identical_to_single_cta(E, coop_env):
    h = E.transmon_resonator_hamiltonian(4, 256).data
    coop_env("1")
    a = E.npad_run(E.HermitianOperator(h), tol=1e-12, max_iter=5000)
    coop_env("0")
    b = E.npad_run(E.HermitianOperator(h), tol=1e-12, max_iter=5000)
    assert a.applied == b.applied == 5000
    np.testing.assert_array_equal(a.current.data, b.current.data)
