"""Experiment runners (experiments.py:233-546) on the GPU
API against the reference runners' own outputs (tests/golden/experiments.npz,
made by oracle/gen_golden.py --only experiments)."""
import ast

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def X():
    from paper_2411_09982_b200 import experiments

    return experiments


@pytest.fixture(scope="module")
def gold():
    from pathlib import Path

    return np.load(Path(__file__).parent / "golden" / "experiments.npz")


CASES = {
    "jch": ("run_jch_mott", "JchMottConfig", {"boundary_npad": 1e-9, "boundary_dense_eig": 1e-12,
                                             "boundary_analytic": 0.0, "rel_err_npad": None,
                                             "rel_err_dense": None}),
    "qubit": ("run_driven_qubit", "DrivenQubitConfig", {}),
    "qubit_sin2": ("run_driven_qubit", "DrivenQubitConfig", {}),
    "chain_traj": ("run_spin_chain", "SpinChainConfig", {}),
    "chain_sweep": ("run_spin_chain", "SpinChainConfig", {"error": 1e-6}),
}


@pytest.mark.parametrize("case", list(CASES))
def test_runner_matches_reference(X, gold, case):
    fn_name, cls_name, tols = CASES[case]
    cfg = X.config_from_dict(getattr(X, cls_name), ast.literal_eval(str(gold[f"{case}__cfg"])))
    fields, rows = getattr(X, fn_name)(cfg)
    for f in fields:
        want = gold[f"{case}__{f}"]
        got = np.array([r[f] for r in rows])
        assert got.shape == want.shape, f
        if want.dtype.kind in "iUSb":
            np.testing.assert_array_equal(got, want, err_msg=f)
            continue
        tol = tols.get(f, 1e-10)
        if tol is None:  # relative errors of tiny numbers: compare absolutely
            np.testing.assert_allclose(got, want, rtol=0, atol=1e-9, err_msg=f)
        elif tol == 0.0:
            np.testing.assert_array_equal(got, want, err_msg=f)
        else:
            np.testing.assert_allclose(got, want, rtol=tol, atol=tol * 1e-3, err_msg=f)


def test_bench_givens_rows(X):
    cfg = X.config_from_dict(X.BenchGivensConfig, {"sizes": [1000, 100000]})
    fields, rows = X.bench_givens(cfg)
    assert [r["dim"] for r in rows] == [1000, 100000]
    for r in rows:
        assert r["nnz"] == 3 * r["dim"] - 3  # the ladder without its zero (0, 0) entry
        assert 0 < r["time_min_s"] <= r["time_median_s"] <= r["time_max_s"]
        assert set(fields) == set(r)


def test_bench_magnus_matched_errors(X):
    # matched-error config (found with the reference runner): errors equal the
    # reference's (magnus 1.1667e-2, rk4 1.8849e-2 at length 4)
    cfg = X.config_from_dict(X.BenchMagnusConfig, {"lengths": [4], "m_magnus": 200, "rk_steps": 200})
    fields, rows = X.bench_magnus(cfg)
    assert [(r["method"], r["length"]) for r in rows] == [("magnus", 4), ("rk4", 4)]
    assert rows[0]["error"] == pytest.approx(0.011666666759862474, rel=1e-8)
    assert rows[1]["error"] == pytest.approx(0.018848689881181702, rel=1e-8)


def test_bench_magnus_unmatched_raises_like_reference(X):
    # the reference's default (m_magnus 20, rk 1000) is not matched at length 4
    from paper_2411_09982_b200.errors import EffHamError

    cfg = X.config_from_dict(X.BenchMagnusConfig, {"lengths": [4]})
    with pytest.raises(EffHamError, match=r"magnus 1\.133e\+00, rk4 3\.034e-05"):
        X.bench_magnus(cfg)


def test_spin_chain_timing_mode(X):
    cfg = X.config_from_dict(X.SpinChainConfig, {"mode": "timing", "lengths": [4], "samples": 4001,
                                                 "rk_steps": 100})
    fields, rows = X.run_spin_chain(cfg)
    assert [r["method"] for r in rows] == ["magnus", "rk4"]
    assert all(r["dim"] == 16 for r in rows)
