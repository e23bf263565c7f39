"""Host-side parts of the drop-in API (no GPU): containers, validation and
error behaviour, builders, closed-form oracles, CSV I/O, the RK4 comparator."""
import numpy as np
import pytest

import paper_2411_09982_b200 as eff


def test_givens_rotation_dataclass_contract():
    r = eff.GivensRotation(0, 3, np.cos(0.3), np.sin(0.3), 0.7)
    u = r.as_matrix(5)
    assert np.allclose(u @ u.conj().T, np.eye(5))
    with pytest.raises(eff.IndexOutOfRange):
        eff.GivensRotation(2, 1, 1.0, 0.0, 0.0)
    with pytest.raises(ValueError):
        eff.GivensRotation(0, 1, 1.0, 0.1, 0.0)
    with pytest.raises(eff.IndexOutOfRange):
        r.as_matrix(3)


def test_hermitian_operator_contract():
    h = np.array([[1.0, 2 - 1j], [2 + 1j, -1.0]])
    op = eff.HermitianOperator(h)
    assert op.dim == 2 and op.layout == "dense"
    h[0, 0] = 99  # copied on construction
    assert op.entry(0, 0) == 1.0
    with pytest.raises(eff.HermiticityViolation):
        eff.HermitianOperator(np.array([[1.0, 1.0], [0.0, 1.0]]))
    with pytest.raises(ValueError):
        eff.HermitianOperator(np.zeros((2, 3)))
    cp = op.largest_couplings(1)[0]
    assert (cp.row, cp.col) == (0, 1) and np.isclose(cp.magnitude, abs(2 + 1j))
    np.testing.assert_array_equal(op.diagonal(), [1.0, -1.0])


def test_control_grid_validation_and_csv(tmp_path):
    with pytest.raises(ValueError):
        eff.ControlGrid(1.0, 0.0, np.zeros((1, 4)))
    with pytest.raises(ValueError):
        eff.ControlGrid(0.0, 1.0, np.array([[0.0, np.nan, 1.0]]))
    g = eff.ControlGrid(0.0, 2.0, np.random.default_rng(0).standard_normal((2, 9)))
    assert g.dt == 0.25 and g.samples == 9
    eff.save_control_grid(g, tmp_path / "g.csv")
    g2 = eff.load_control_grid(tmp_path / "g.csv")
    np.testing.assert_array_equal(g2.signals, g.signals)
    with pytest.raises(eff.GridMismatch):
        g.with_signals(np.zeros((2, 5)))


def test_transmon_resonator_builder():
    op = eff.transmon_resonator_hamiltonian(3, 20)
    h = op.data
    assert h.shape == (60, 60)
    np.testing.assert_array_equal(h, h.conj().T)
    # diagonal: wq q + a/2 q(q-1) + wr n ; coupling g sqrt(q+1) sqrt(n+1)
    assert np.isclose(h[1 * 20 + 3, 1 * 20 + 3].real, 5.0 + 7.0 * 3)
    assert np.isclose(h[0 * 20 + 0, 1 * 20 + 1].real, 0.1)
    assert np.isclose(h[1 * 20 + 2, 2 * 20 + 3].real, 0.1 * np.sqrt(2) * np.sqrt(3))
    pts = eff.sweep_points()
    assert pts.shape == (1024, 4)
    assert eff.sweep_target(256) == [0, 1, 2, 3, 4, 256, 257, 258, 259, 260]


def test_heisenberg_chain_builder():
    ch = eff.heisenberg_chain_hamiltonians(6)
    h0 = ch.drift.to_dense()
    np.testing.assert_allclose(h0, h0.conj().T)
    # total magnetisation conserved by XX+YY+ZZ: commutes with sum Z
    z = np.diag([sum(1 - 2 * ((x >> j) & 1) for j in range(6)) for x in range(64)]).astype(complex)
    assert np.abs(h0 @ z - z @ h0).max() < 1e-12
    # ferromagnetic state energy = J * L
    assert np.isclose(h0[0, 0].real, 6.0)


def test_closed_forms():
    p = eff.JCSiteParams(omega=1.0, qubit_freq=0.9, g=0.05, n_max=6)
    lo, hi = eff.jc_doublet_energies(p, 2)
    blk = eff.jc_onsite_hamiltonian(p).to_dense()[3:5, 3:5]
    w = np.linalg.eigvalsh(blk)
    assert np.allclose([lo, hi], w, atol=1e-13)
    for n in (1, 2, 3):
        for x in (-1.0, 0.3):
            q = eff.JCSiteParams(omega=1.0, qubit_freq=1.0 - x * 0.1, g=0.1, mu=0.0, n_max=8)
            assert abs(eff.mott_lobe_boundary_dense(q, n) - eff.mott_lobe_boundary_analytic(n, x)) < 1e-9


def test_rk4_comparator_argument_checks():
    # validated on the host before any device work (numerics: tests/test_rk4_gpu.py)
    h = np.array([[0.3, 0.1], [0.1, -0.2]], dtype=complex)
    ch = eff.ControlledHamiltonian(eff.HermitianOperator(h))
    grid = eff.ControlGrid(0.0, 1.0, samples=401)
    with pytest.raises(eff.GridMismatch):
        eff.rk4_evolve(ch, grid, 3, np.array([1, 0], dtype=complex))
    with pytest.raises(eff.GridMismatch):
        eff.rk4_evolve(ch, grid, 0, np.array([1, 0], dtype=complex))
    with pytest.raises(eff.DimensionMismatch):
        eff.rk4_evolve(ch, grid, 200, np.array([1, 0, 0], dtype=complex))


def test_infidelity_and_states():
    a = np.array([1, 0], dtype=complex)
    b = np.array([1, 1], dtype=complex) / np.sqrt(2)
    assert np.isclose(eff.infidelity(a, b), 0.5)
    with pytest.raises(eff.DimensionMismatch):
        eff.infidelity(a, np.array([1, 0, 0], dtype=complex))
    with pytest.raises(ValueError):
        eff.StateVector([1.0, 1.0])


def test_experiment_configs_validate():
    from paper_2411_09982_b200 import errors, experiments as X

    with pytest.raises(errors.ConfigError):
        X.config_from_dict(X.JchMottConfig, {"bogus": 1})
    with pytest.raises(errors.ConfigError):
        X.config_from_dict(X.DrivenQubitConfig, {"m_magnus": 7})
    with pytest.raises(errors.ConfigError):
        X.config_from_dict(X.SpinChainConfig, {"mode": "timing", "repeats": 2})
    cfg = X.config_from_dict(X.SpinChainConfig, {"mode": "error-sweep"})
    assert cfg.samples == 16001
    assert X.relative_error(1.0, 0.0) == 1.0 / 1e-300
    assert X.state_distance([1, 0], [0, 1]) == pytest.approx(np.sqrt(2))


def test_experiment_csv(tmp_path):
    from paper_2411_09982_b200 import experiments as X

    p = tmp_path / "out.csv"
    X.write_csv(p, ["a", "b"], [{"a": 1, "b": 0.1}, {"a": 2, "b": 1e-300}])
    assert p.read_text() == "a,b\n1,0.1\n2,1e-300\n"
