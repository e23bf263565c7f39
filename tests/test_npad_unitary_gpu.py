"""Accumulated-unitary tracking (npad.py:244-259) on the paths the first
round left thin: the whole-GPU chain (dim >= 1024) with U rows updated in
the cluster kernel and the audit pauses every 100 rotations; the
UnitarityDrift audit of eliminate_couplings at exactly the multiples of 100
the reference checks (npad.py:290-296); sparse operators with U tracking stay
sparse.  Bars: pivots bit-exact, matrices 1e-10 relative."""
import numpy as np
import pytest

from conftest import rel_fro
from oracle import npad_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    import paper_2411_09982_b200 as eff

    return eff


@pytest.mark.parametrize("k", [99, 100, 250])
def test_track_unitary_whole_gpu_chain_vs_oracle(E, k):
    h = E.transmon_resonator_hamiltonian(4, 256).data  # dim 1024: the cluster driver
    ref = npad_oracle.run_incremental(h, tol=1e-12, max_iter=k, track_unitary=True)
    st, piv = E.npad_run_logged(E.HermitianOperator(h), tol=1e-12, max_iter=k, track_unitary=True)
    assert st.applied == ref["applied"] == k and not st.converged
    np.testing.assert_array_equal(piv, ref["pivots"])
    assert rel_fro(st.current.data, ref["h"]) <= 1e-10
    assert rel_fro(st.accumulated_unitary, ref["u"]) <= 1e-10


def test_track_unitary_timing_not_single_cta(E):
    # dim 4096 with U: the cluster kernel (rows of U on the CTAs' columns) —
    # 300 rotations (3 audits) well under a second
    import time

    h = E.transmon_resonator_hamiltonian(4, 1024).data
    op = E.HermitianOperator(h, validate=False)
    E.npad_run(op, tol=1e-12, max_iter=10, track_unitary=True)
    t0 = time.perf_counter()
    st = E.npad_run(op, tol=1e-12, max_iter=300, track_unitary=True)
    dt = time.perf_counter() - t0
    assert st.applied == 300
    assert dt < 2.0, dt
    u = st.accumulated_unitary
    assert np.linalg.norm(u @ u.conj().T - np.eye(u.shape[0])) <= 1e-10 * u.shape[0]


def test_eliminate_couplings_audits_at_multiples_of_100(E):
    # a drifted U: the reference raises right after the rotation that makes
    # applied == 100, with that count in the message
    h = E.transmon_resonator_hamiltonian(3, 20).data
    op = E.HermitianOperator(h)
    pairs = [(0, 21), (1, 22), (2, 23), (3, 24)]
    u_bad = np.eye(60, dtype=complex) * (1.0 + 1e-6)
    ok = E.NPADState(current=op, applied=90, accumulated_unitary=u_bad.copy())
    E.eliminate_couplings(ok, pairs)  # 91..94: no audit point
    st = E.NPADState(current=op, applied=98, accumulated_unitary=u_bad.copy())
    with pytest.raises(E.UnitarityDrift, match="after 100 rotations"):
        E.eliminate_couplings(st, pairs)
    # a good U through an audit point: same result as one segment
    good = E.NPADState(current=op, applied=98, accumulated_unitary=np.eye(60, dtype=complex))
    out = E.eliminate_couplings(good, pairs)
    hr, ur = npad_oracle.eliminate_pairs(h, pairs, np.eye(60, dtype=complex))
    assert out.applied == 102
    assert rel_fro(out.current.data, hr) <= 1e-12 and rel_fro(out.accumulated_unitary, ur) <= 1e-12


def test_sparse_operator_with_unitary_stays_sparse(E, golden):
    import scipy.sparse as sps

    g = golden("npad_sparse")
    n = len(g["rnd_indptr"]) - 1
    m = sps.csr_matrix((g["rnd_data"], g["rnd_indices"], g["rnd_indptr"]), shape=(n, n))
    op = E.HermitianOperator(m)
    st0 = E.NPADState.from_operator(op, track_unitary=True)
    dense = m.toarray()
    pairs = [(int(a), int(b)) for a, b in g["rnd_pivots"][:1]]
    out = E.eliminate_couplings(st0, pairs)
    assert out.current.layout == "sparse"
    hr, ur = npad_oracle.eliminate_pairs(dense, pairs, np.eye(n, dtype=complex))
    assert rel_fro(out.current.to_dense(), hr) <= 1e-12
    assert rel_fro(out.accumulated_unitary, ur) <= 1e-12
