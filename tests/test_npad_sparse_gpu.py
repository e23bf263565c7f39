"""Sparse CSR Givens rotations on the device (npad_sparse.cu) — the
reference's _conjugate_sparse (npad.py:148-232) and the paper's bench_givens
protocol (experiments.py:420-453) — against golden vectors of the reference
itself and the oracle restatement: same CSR structure, same bits."""
import numpy as np
import pytest
import scipy.sparse as sps

from oracle import npad_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    import paper_2411_09982_b200 as eff

    return eff


def _csr(g, p, n):
    return sps.csr_matrix((g[p + "_data"], g[p + "_indices"], g[p + "_indptr"]), shape=(n, n))


def _same(a, b):
    a = a.tocsr()
    np.testing.assert_array_equal(a.indptr, b.indptr)
    np.testing.assert_array_equal(a.indices, b.indices)
    np.testing.assert_array_equal(a.data, b.data)


def test_ladder_bench_rotation_golden(E, golden):
    g = golden("npad_sparse")
    n = g["lad_indptr"].size - 1
    op = E.HermitianOperator(_csr(g, "lad", n), validate=False)
    st = E.eliminate_coupling(E.NPADState.from_operator(op), 0, 1)
    assert st.current.layout == "sparse" and st.applied == 1
    _same(st.current.data, _csr(g, "lad_out", n))


def test_sparse_chain_replay_golden(E, golden):
    # the reference's sparse npad_run (40 greedy rotations): replay its pivots
    g = golden("npad_sparse")
    n = g["rnd_indptr"].size - 1
    st = E.NPADState.from_operator(E.HermitianOperator(_csr(g, "rnd", n)))
    for i, j in g["rnd_pivots"]:
        st = E.eliminate_coupling(st, int(i), int(j))
    _same(st.current.data, _csr(g, "rnd_out", n))
    assert st.current.max_abs() == float(np.max(np.abs(g["rnd_out_data"])))


def test_fill_in_drop_golden(E, golden):
    g = golden("npad_sparse")
    op = E.HermitianOperator(sps.csr_matrix(g["can_dense"]), validate=False)
    st = E.eliminate_coupling(E.NPADState.from_operator(op), 0, 1)
    _same(st.current.data, _csr(g, "can_out", 3))


def test_rotation_errors(E, golden):
    g = golden("npad_sparse")
    n = g["lad_indptr"].size - 1
    op = E.HermitianOperator(_csr(g, "lad", n), validate=False)
    with pytest.raises(E.ZeroCoupling):
        E.eliminate_coupling(E.NPADState.from_operator(op), 0, 5)
    with pytest.raises(E.IndexOutOfRange):
        E.eliminate_coupling(E.NPADState.from_operator(op), 1, n)


@pytest.mark.parametrize("n", [10**5, 10**6])
def test_ladder_full_size_vs_oracle(E, n):
    # bench_givens sizes: one rotation on the ladder a^dag a + (a + a^dag)
    op = E.ladder_test_hamiltonian(n)
    st = E.eliminate_coupling(E.NPADState.from_operator(op), 0, 1)
    ref = npad_oracle.eliminate_sparse(op.data, 0, 1)
    _same(st.current.data, ref)


def test_eliminate_couplings_sparse_jc(E):
    # Mott-lobe pairs on the sparse JC site (models.py:112-131) vs the oracle
    p = E.JCSiteParams(omega=1.0, qubit_freq=0.8, g=0.1, mu=0.3, n_max=8)
    op = E.jc_onsite_hamiltonian(p)
    assert op.layout == "sparse"
    pairs = [(2 * m - 1, 2 * m) for m in range(1, 6)]
    st = E.eliminate_couplings(E.NPADState.from_operator(op), pairs)
    m = op.data.tocsr()
    rots = [npad_oracle.sparse_rotation_scalars(m, i, j) for i, j in pairs]
    mx = m
    for (i, j), (ch, sh, ph, _) in zip(pairs, rots):
        mx = npad_oracle.conjugate_sparse(mx, i, j, ch, sh, ph, float(np.max(np.abs(mx.data))))
    _same(st.current.data, mx)


def test_device_ladder_builder(E):
    for n in (2, 3, 1000, 100_001):
        dev = E.ladder_test_hamiltonian_device(n)
        _same(dev.data, E.ladder_test_hamiltonian(n).data)
        assert dev.max_abs() == E.ladder_test_hamiltonian(n).max_abs()


def test_sparse_npad_run_golden(E, golden):
    # the reference's npad_run on a sparse operator, 40 greedy rotations:
    # same pivots, same sparse result
    g = golden("npad_sparse")
    n = g["rnd_indptr"].size - 1
    op = E.HermitianOperator(_csr(g, "rnd", n))
    st, piv = E.npad_run_logged(op, tol=1e-12, max_iter=40)
    assert st.current.layout == "sparse" and st.applied == 40 and not st.converged
    np.testing.assert_array_equal(piv, g["rnd_pivots"])
    _same(st.current.data, _csr(g, "rnd_out", n))


@pytest.mark.parametrize("target", [None, [0, 3, 7], []])
def test_sparse_npad_run_vs_oracle_to_convergence(E, target):
    # sparse JC lattice-like operator: greedy chain to convergence vs the oracle
    p = E.JCSiteParams(omega=1.0, qubit_freq=0.8, g=0.1, mu=0.3, n_max=10)
    op = E.jc_onsite_hamiltonian(p)
    m = op.data.tocsr()
    st, piv = E.npad_run_logged(op, target, tol=1e-12)
    # oracle: reference selection on the CSR, reference sparse rotation
    thr = 1e-12 * float(np.max(np.abs(m.data)))
    ref_piv = []
    while True:
        low = sps.tril(m, k=-1, format="coo")
        r, c, v = low.row, low.col, low.data
        keep = v != 0
        if target is not None:
            ts = np.asarray(sorted(target), dtype=np.int64)
            keep &= np.isin(r, ts) ^ np.isin(c, ts)
        r, c, v = r[keep], c[keep], v[keep]
        if r.size == 0:
            break
        mags = np.abs(v)
        k = np.lexsort((r, c, -mags))[0]
        if mags[k] < thr:
            break
        ref_piv.append((int(c[k]), int(r[k])))
        m = npad_oracle.eliminate_sparse(m, int(c[k]), int(r[k]))
    assert st.converged
    np.testing.assert_array_equal(piv.reshape(-1, 2), np.asarray(ref_piv, dtype=np.int32).reshape(-1, 2))
    _same(st.current.data, m)
