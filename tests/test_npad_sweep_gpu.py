"""The many-chain subspace drivers (npad_warp.cu, npad_cta.cu: lazy
columns) — the BASELINE config-4 sweep path — against the oracle and against
the eager block driver, bit for bit."""
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


@pytest.fixture(params=["cta", "warp", "tsmem"])
def warp_mode(request):
    """Force a many-chain driver (npad_cta.cu / npad_warp.cu / npad_tsmem.cu)
    even for one chain."""
    old = os.environ.get("QCH_NPAD_DRIVER")
    os.environ["QCH_NPAD_DRIVER"] = request.param
    yield request.param
    if old is None:
        del os.environ["QCH_NPAD_DRIVER"]
    else:
        os.environ["QCH_NPAD_DRIVER"] = old


def _herm(n, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    h = (a + a.conj().T) * (0.5 * scale)
    h = np.triu(h) + np.triu(h, 1).conj().T  # bitwise Hermitian
    return h + np.diag(np.arange(n, dtype=float))


def test_warp_driver_golden_subspace(E, golden, warp_mode):
    g = golden("npad_tr4x30_sub")
    st, piv = E.npad_run_logged(E.HermitianOperator(g["h"]), g["target"].tolist(), tol=float(g["tol"]))
    np.testing.assert_array_equal(piv, g["pivots"])
    assert st.applied == int(g["applied"]) and st.converged == bool(g["converged"])
    assert rel_fro(st.current.data, g["final"]) <= TOL_F


@pytest.mark.parametrize("n,nt,seed", [(40, 3, 1), (150, 10, 2), (257, 32, 3)])
def test_warp_driver_random_vs_oracle(E, warp_mode, n, nt, seed):
    h = _herm(n, seed)
    tgt = sorted(np.random.default_rng(seed + 100).choice(n, nt, replace=False).tolist())
    ref = npad_oracle.run_incremental(h, tgt, tol=1e-12)
    st, piv = E.npad_run_logged(E.HermitianOperator(h), tgt, tol=1e-12)
    np.testing.assert_array_equal(piv, ref["pivots"])
    assert st.applied == ref["applied"] and st.converged == ref["converged"]
    assert rel_fro(st.current.data, ref["h"]) <= TOL_F


def test_driver_many_touched_rows(E, warp_mode):
    # a dense chain that touches far more than 128 distinct rows: exercises the
    # mid-chain column flush of the lazy scheme
    n = 420
    h = _herm(n, 7, scale=0.3)
    tgt = list(range(0, n, 35))  # 12 target levels spread over the spectrum
    ref = npad_oracle.run_incremental(h, tgt, tol=1e-12, max_iter=2500)
    assert len(set(ref["pivots"].ravel().tolist())) > 140
    st, piv = E.npad_run_logged(E.HermitianOperator(h), tgt, tol=1e-12, max_iter=2500)
    np.testing.assert_array_equal(piv, ref["pivots"])
    assert rel_fro(st.current.data, ref["h"]) <= TOL_F


def test_lazy_columns_bit_identical_to_eager(E):
    # batch (warp driver, lazy columns) vs single runs (block driver, eager
    # mirrored columns): the same matrices, bit for bit
    pts = E.sweep_points(4, 4)[[0, 5, 10, 15]]
    nq, nr = 4, 64
    tgt = E.sweep_target(nr)
    res = E.npad_sweep_transmon(pts, nq, nr, tgt, tol=1e-12)
    old = os.environ.get("QCH_NPAD_DRIVER")
    os.environ["QCH_NPAD_DRIVER"] = "block"
    try:
        for b, row in enumerate(pts):
            h = E.transmon_resonator_hamiltonian(nq, nr, omega_q=row[0], alpha=row[1], omega_r=row[2], g=row[3]).data
            st = E.npad_run(E.HermitianOperator(h), tgt, tol=1e-12)
            assert st.applied == res.applied[b]
            np.testing.assert_array_equal(res.operator(b).data, st.current.data)
    finally:
        if old is None:
            del os.environ["QCH_NPAD_DRIVER"]
        else:
            os.environ["QCH_NPAD_DRIVER"] = old


def test_config4_sweep_full_size(E):
    # BASELINE config 4: 1024 (g, Delta) points of a dim-1024 transmon x
    # resonator, subspace target of 10 levels; sampled points vs the oracle,
    # size-independent properties on all of them
    import torch

    nq, nr = 4, 256
    pts = E.sweep_points(32, 32)
    tgt = E.sweep_target(nr)
    res = E.npad_sweep_transmon(pts, nq, nr, tgt, tol=1e-12)
    assert bool(np.all(res.converged))
    assert 300_000 < int(np.sum(res.applied)) < 600_000
    for b in (0, 31, 512, 700, 1023):
        row = pts[b]
        h = E.transmon_resonator_hamiltonian(nq, nr, omega_q=row[0], alpha=row[1], omega_r=row[2], g=row[3]).data
        ref = npad_oracle.run_incremental(h, tgt, tol=1e-12)
        assert res.applied[b] == ref["applied"]
        assert rel_fro(res.operator(b).data, ref["h"]) <= TOL_F
    # every output is bitwise Hermitian and keeps its trace
    mats = res.matrices if hasattr(res, "matrices") else None
    if mats is not None:
        for b in range(0, 1024, 97):
            m = mats[b]
            assert bool(torch.equal(m, m.conj().T))


@pytest.mark.parametrize("handover", ["40", "0", "1000"])
def test_sweep_handover_to_shared_memory_driver(E, handover):
    # 200 sweep points (dim 256): the warp driver runs every chain until
    # <= handover are left, the T-rows-in-shared-memory driver finishes them
    # (0: warp driver only; 1000: shared-memory driver from the start) — the
    # same per-point results as npad_run on each operator, matrices bit for bit
    old = os.environ.get("QCH_NPAD_HANDOVER")
    os.environ["QCH_NPAD_HANDOVER"] = handover
    try:
        nq, nr = 4, 64
        pts = E.sweep_points(20, 10)
        tgt = E.sweep_target(nr)
        res = E.npad_sweep_transmon(pts, nq, nr, tgt, tol=1e-12)
    finally:
        if old is None:
            del os.environ["QCH_NPAD_HANDOVER"]
        else:
            os.environ["QCH_NPAD_HANDOVER"] = old
    assert res.converged.all()
    for k in (0, 57, 133, 199):
        wq, al, wr, g = pts[k]
        h = E.transmon_resonator_hamiltonian(nq, nr, omega_q=wq, alpha=al, omega_r=wr, g=g).data
        ref = npad_oracle.run_incremental(h, tgt, tol=1e-12)
        assert int(res.applied[k]) == ref["applied"]
        assert rel_fro(res.operator(k).data, ref["h"]) <= TOL_F
        single = E.npad_run(E.HermitianOperator(h), tgt, tol=1e-12)
        np.testing.assert_array_equal(res.operator(k).data, single.current.data)
