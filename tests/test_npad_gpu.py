"""NPAD on the GPU vs the oracle / golden vectors (parity gate).

Bar (north star): bit-exact pivot sequence, applied count and converged
flag; <= 1e-10 relative Frobenius error on matrices; eigen/diagonal values
to 1e-10 relative."""
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


def _run(E, h, target=None, **kw):
    return E.npad_run_logged(E.HermitianOperator(h), target, **kw)


@pytest.mark.parametrize("case", ["npad_tr3x20_full", "npad_rand24_full_u", "npad_tr4x30_sub", "npad_tr4x60_k150"])
def test_npad_run_matches_reference_golden(E, golden, case):
    g = golden(case)
    target = g["target"].tolist() if "target" in g else None
    max_iter = int(g["max_iter"]) if "max_iter" in g else None
    st, piv = _run(E, g["h"], target, tol=float(g["tol"]), max_iter=max_iter, track_unitary="u" in g)
    assert st.applied == int(g["applied"])
    assert st.converged == bool(g["converged"])
    np.testing.assert_array_equal(piv, g["pivots"])
    assert rel_fro(st.current.data, g["final"]) <= TOL_F
    if "u" in g:
        assert rel_fro(st.accumulated_unitary, g["u"]) <= TOL_F


def test_npad_run_api_object(E, golden):
    g = golden("npad_tr3x20_full")
    st = E.npad_run(E.HermitianOperator(g["h"]), tol=1e-12)
    assert isinstance(st, E.NPADState)
    assert st.applied == 1022 and st.converged
    d = st.current.diagonal()
    np.testing.assert_allclose(np.sort(d), np.sort(np.linalg.eigvalsh(g["h"])), rtol=1e-10, atol=1e-10)


@pytest.mark.parametrize("n,seed", [(2, 1), (5, 2), (31, 3), (64, 4), (113, 5), (150, 6)])
def test_npad_random_hermitian_vs_oracle(E, n, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    h = (a + a.conj().T) / 2
    ref = npad_oracle.run_incremental(h, tol=1e-12, max_iter=3000)
    st, piv = _run(E, h, tol=1e-12, max_iter=3000)
    np.testing.assert_array_equal(piv, ref["pivots"])
    assert st.applied == ref["applied"] and st.converged == ref["converged"]
    assert rel_fro(st.current.data, ref["h"]) <= TOL_F


@pytest.mark.parametrize("nq,nr,target", [(3, 20, [0, 1, 20, 21]), (4, 64, list(range(5)) + list(range(64, 69))),
                                          (2, 40, [])])
def test_npad_subspace_vs_oracle(E, nq, nr, target):
    h = E.transmon_resonator_hamiltonian(nq, nr, omega_q=6.1, g=0.12).data
    ref = npad_oracle.run_incremental(h, target, tol=1e-12)
    st, piv = _run(E, h, target, tol=1e-12)
    np.testing.assert_array_equal(piv, ref["pivots"])
    assert st.applied == ref["applied"] and st.converged == ref["converged"]
    assert rel_fro(st.current.data, ref["h"]) <= TOL_F


def test_npad_large_truncated_vs_oracle(E):
    # dim 1024 (4 x 256), first 400 rotations: global-memory driver
    h = E.transmon_resonator_hamiltonian(4, 256).data
    ref = npad_oracle.run_incremental(h, tol=1e-12, max_iter=400)
    st, piv = _run(E, h, tol=1e-12, max_iter=400)
    assert st.applied == 400 and not st.converged
    np.testing.assert_array_equal(piv, ref["pivots"])
    assert rel_fro(st.current.data, ref["h"]) <= TOL_F


def test_npad_not_bitwise_hermitian_input(E):
    # Hermitian to 1e-15 but not bitwise: exercises the column-reading path
    rng = np.random.default_rng(9)
    a = rng.standard_normal((20, 20)) + 1j * rng.standard_normal((20, 20))
    h = (a + a.conj().T) / 2
    h = h + 1e-15 * (rng.standard_normal((20, 20)))
    ref = npad_oracle.run_full_scan(h, tol=1e-12, max_iter=500)
    st, piv = _run(E, h, tol=1e-12, max_iter=500)
    np.testing.assert_array_equal(piv, ref["pivots"])
    assert rel_fro(st.current.data, ref["h"]) <= TOL_F


def test_npad_edge_cases(E):
    st = E.npad_run(E.HermitianOperator(np.array([[3.0]])), tol=1e-12)
    assert st.applied == 0 and st.converged
    st = E.npad_run(E.HermitianOperator(np.zeros((5, 5))), tol=1e-12)
    assert st.applied == 0 and st.converged
    st = E.npad_run(E.HermitianOperator(np.diag([1.0, 2.0, 3.0])), tol=1e-12)
    assert st.applied == 0 and st.converged
    h = E.transmon_resonator_hamiltonian(3, 20).data
    st = E.npad_run(E.HermitianOperator(h), tol=1e-12, max_iter=0)
    assert st.applied == 0 and not st.converged
    with pytest.raises(ValueError):
        E.npad_run(E.HermitianOperator(h), tol=0.0)
    with pytest.raises(E.IndexOutOfRange):
        E.npad_run(E.HermitianOperator(h), [60], tol=1e-12)


def test_givens_and_unitary_transformation(E, golden):
    g = golden("givens_2x2")
    for k in range(0, 1000, 10):
        op = E.HermitianOperator(g["mats"][k])
        rot = E.givens_rotation_matrix(op, 0, 1)
        c, sh, ph, deg = g["params"][k]
        assert abs(rot.cos_half - c) <= 4e-16 and abs(rot.sin_half - sh) <= 4e-16
        assert rot.degenerate == bool(deg)
        new = E.unitary_transformation(op, rot)
        assert rel_fro(new.data, g["after"][k]) <= 1e-14
        # AC1: off-diagonal annihilated, ordering preserved
        assert abs(new.data[1, 0]) <= 1e-13 * np.abs(g["mats"][k]).max()
    with pytest.raises(E.ZeroCoupling):
        E.givens_rotation_matrix(E.HermitianOperator(np.diag([1.0, 2.0])), 0, 1)
    with pytest.raises(E.IndexOutOfRange):
        E.givens_rotation_matrix(E.HermitianOperator(np.eye(3)), 2, 1)


def test_eliminate_couplings_fused(E, golden):
    g = golden("npad_jc_pairs")
    st0 = E.NPADState.from_operator(E.HermitianOperator(g["h"]), track_unitary=True)
    st = E.eliminate_couplings(st0, [tuple(p) for p in g["pairs"]])
    assert st.applied == int(g["applied"])
    assert rel_fro(st.current.data, g["final"]) <= 1e-14
    assert rel_fro(st.accumulated_unitary, g["u"]) <= 1e-14
    with pytest.raises(E.OverlappingPairs):
        E.eliminate_couplings(st0, [(1, 2), (2, 3)])
    assert E.eliminate_couplings(st0, []) is st0


def test_eliminate_couplings_cross_terms_vs_oracle(E):
    rng = np.random.default_rng(5)
    a = rng.standard_normal((40, 40)) + 1j * rng.standard_normal((40, 40))
    h = (a + a.conj().T) / 2
    pairs = [(3, 17), (0, 39), (5, 6), (20, 30)]
    ref, _ = npad_oracle.eliminate_pairs(h, pairs)
    st = E.eliminate_couplings(E.NPADState.from_operator(E.HermitianOperator(h)), pairs)
    assert rel_fro(st.current.data, ref) <= 1e-14


def test_mott_lobes_npad_vs_analytic(E):
    # SPEC AC3 (subset): NPAD boundaries vs Eq. 8
    for n in (1, 3):
        for x in (-2.0, -0.5, 0.0, 1.25):
            g = 0.1
            p = E.JCSiteParams(omega=1.0, qubit_freq=1.0 - x * g, g=g, mu=0.2, n_max=8)
            got = E.mott_lobe_boundary_npad(p, n)
            want = E.mott_lobe_boundary_analytic(n, x)
            assert abs(got - want) <= 1e-9 * max(1.0, abs(want))


def test_batch_sweep_matches_single_runs(E):
    pts = E.sweep_points(3, 3, omega_r=7.0)
    nq, nr = 4, 40
    tgt = E.sweep_target(nr)
    res = E.npad_sweep_transmon(pts, nq, nr, tgt, tol=1e-12)
    for b, row in enumerate(pts):
        h = E.transmon_resonator_hamiltonian(nq, nr, omega_q=row[0], alpha=row[1], omega_r=row[2], g=row[3]).data
        ref = npad_oracle.run_incremental(h, tgt, tol=1e-12)
        assert res.applied[b] == ref["applied"] and res.converged[b] == ref["converged"]
        assert rel_fro(res.operator(b).data, ref["h"]) <= TOL_F


def test_device_builder_matches_host(E):
    import torch

    pts = E.sweep_points(2, 2)
    mats = E.npad.build_transmon_resonator_batch(pts, 4, 16)
    for b, row in enumerate(pts):
        h = E.transmon_resonator_hamiltonian(4, 16, omega_q=row[0], alpha=row[1], omega_r=row[2], g=row[3]).data
        np.testing.assert_array_equal(mats[b].cpu().numpy(), h)
