"""NPAD at the BASELINE sizes against the REFERENCE ITSELF (golden vectors
made by running effham: oracle/gen_golden.py --only large): config-4 sweep
points (dim 1024, subspace mode, to convergence) through the single-chain,
batched and device-built sweep paths, and the first 60 rotations of config 3
(dim 4096, full mode) through the whole-GPU cluster driver."""
from pathlib import Path

import numpy as np
import pytest

from conftest import rel_fro

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def E():
    import paper_2411_09982_b200 as eff

    return eff


@pytest.fixture(scope="module")
def G():
    return np.load(Path(__file__).parent / "golden" / "npad_large_ref.npz")


def _sweep_h(E, pt):
    wq, al, wr, g = pt
    return E.transmon_resonator_hamiltonian(4, 256, omega_q=wq, alpha=al, omega_r=wr, g=g).data


@pytest.mark.parametrize("k", [0, 1, 2])
def test_sweep_point_single_chain(E, G, k):
    h = _sweep_h(E, G[f"sweep{k}_point"])
    tgt = E.sweep_target(256)
    want = G[f"sweep{k}_pivots"]
    st, piv = E.npad_run_logged(E.HermitianOperator(h), tgt, tol=1e-12, pivot_cap=len(want))
    assert st.applied == int(G[f"sweep{k}_applied"]) and st.converged == bool(G[f"sweep{k}_converged"])
    np.testing.assert_array_equal(piv, want)
    fin = st.current.data
    assert rel_fro(np.real(np.diag(fin)), G[f"sweep{k}_diag"]) <= TOL
    assert rel_fro(fin[[0, 4, 256, 700]], G[f"sweep{k}_rows"]) <= TOL


def test_sweep_points_batched_and_device_built(E, G):
    tgt = E.sweep_target(256)
    pts = np.stack([G[f"sweep{k}_point"] for k in range(3)])
    res = E.npad_run_batch([E.HermitianOperator(_sweep_h(E, p)) for p in pts], tgt, tol=1e-12)
    dev = E.npad_sweep_transmon(pts, 4, 256, tgt, tol=1e-12)
    for k in range(3):
        for r in (res, dev):
            assert int(r.applied[k]) == int(G[f"sweep{k}_applied"])
            fin = r.operator(k).data
            assert rel_fro(np.real(np.diag(fin)), G[f"sweep{k}_diag"]) <= TOL
            assert rel_fro(fin[[0, 4, 256, 700]], G[f"sweep{k}_rows"]) <= TOL


def test_config3_first_rotations(E, G):
    h = E.transmon_resonator_hamiltonian(4, 1024).data
    want = G["c3_pivots"]
    st, piv = E.npad_run_logged(E.HermitianOperator(h), tol=1e-12, max_iter=int(G["c3_applied"]))
    assert st.applied == int(G["c3_applied"]) and not st.converged
    np.testing.assert_array_equal(piv, want)
    fin = st.current.data
    assert rel_fro(np.real(np.diag(fin)), G["c3_diag"]) <= TOL
    assert rel_fro(fin[G["c3_rows_idx"]], G["c3_rows"]) <= TOL


def test_config3_full_length_vs_oracle(E, G):
    # BASELINE config 3 to convergence: all 292,068 greedy picks bit-equal to
    # the oracle (npad_oracle.run_incremental, itself bit-identical to the
    # reference on the first 60 picks above and on every case the reference
    # can finish; oracle/gen_golden_long.py), final diagonal and rows <= 1e-10
    L = np.load(Path(__file__).parent / "golden" / "npad_config3_full_oracle.npz")
    want = L["pivots"].astype(np.int64)
    h = E.transmon_resonator_hamiltonian(4, 1024).data
    st, piv = E.npad_run_logged(E.HermitianOperator(h), tol=1e-12, pivot_cap=len(want) + 16)
    assert st.applied == int(L["applied"]) == len(want) and st.converged == bool(L["converged"])
    bad = np.flatnonzero((piv != want).any(axis=1)) if piv.shape == want.shape else [-1]
    assert len(bad) == 0, f"first differing pick at rotation {bad[0]} of {len(want)}"
    fin = st.current.data
    assert rel_fro(np.real(np.diag(fin)), L["diag"]) <= TOL
    assert rel_fro(fin[L["rows_idx"]], L["rows"]) <= TOL
