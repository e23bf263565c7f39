"""The RK4 comparator on the GPU (reference.py:11-65) against a numpy
restatement of the reference loop and against closed forms."""
import numpy as np
import pytest

from conftest import rel_fro

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    import paper_2411_09982_b200 as eff

    return eff


def _rk4_numpy(ops, signals, t0, t1, steps, psi0):
    """reference.py:11-65 statement by statement (dense numpy)."""
    total = signals.shape[1] - 1
    stride = total // steps
    h = (t1 - t0) / steps

    def ham(idx):
        m = ops[0]
        for k in range(1, len(ops)):
            m = m + signals[k - 1, idx] * ops[k]
        return m

    psi = psi0.astype(complex).copy()
    out = [psi]
    lo = ham(0)
    for n in range(steps):
        mid, hi = ham(n * stride + stride // 2), ham((n + 1) * stride)
        k1 = -1j * (lo @ psi)
        k2 = -1j * (mid @ (psi + (h / 2.0) * k1))
        k3 = -1j * (mid @ (psi + (h / 2.0) * k2))
        k4 = -1j * (hi @ (psi + h * k3))
        psi = psi + (h / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
        out.append(psi)
        lo = hi
    return np.array(out)


def test_constant_hamiltonian_closed_form(E):
    h = np.array([[0.3, 0.1], [0.1, -0.2]], dtype=complex)
    ch = E.ControlledHamiltonian(E.HermitianOperator(h))
    grid = E.ControlGrid(0.0, 1.0, samples=401)
    tr = E.rk4_evolve(ch, grid, 200, np.array([1, 0], dtype=complex))
    w, v = np.linalg.eigh(h)
    exact = v @ (np.exp(-1j * w) * (v.conj().T @ np.array([1, 0])))
    assert np.linalg.norm(tr.amplitudes[-1] - exact) < 1e-10
    np.testing.assert_array_equal(tr.times, np.linspace(0.0, 1.0, 201))


@pytest.mark.parametrize("length,steps", [(4, 100), (6, 250), (9, 50)])
def test_spin_chain_vs_numpy_restatement(E, length, steps):
    ch = E.spin_chain_hamiltonians(E.SpinChainParams(length, 0.3, 0.5, 0.2))
    grid = E.synthetic_transfer_pulse(5.0, 1001, 7)
    psi0 = np.zeros(ch.dim, dtype=complex)
    psi0[0] = 1
    got = E.rk4_evolve(ch, grid, steps, psi0).amplitudes
    ops = [ch.drift.to_dense()] + [c.to_dense() for c in ch.controls]
    want = _rk4_numpy(ops, grid.signals, grid.t_start, grid.t_end, steps, psi0)
    assert rel_fro(got, want) <= 1e-12


def test_large_chain_multi_cta(E):
    # 2^12 states: enough stored entries for the cooperative multi-CTA path
    ch = E.spin_chain_hamiltonians(E.SpinChainParams(12, 0.0, 0.5, 0.2))
    grid = E.synthetic_transfer_pulse(2.0, 401, 3)
    psi0 = np.zeros(ch.dim, dtype=complex)
    psi0[5] = 1
    got = E.rk4_evolve(ch, grid, 40, psi0).amplitudes
    ops = [ch.drift.data.tocsr()] + [c.data.tocsr() for c in ch.controls]
    want = _rk4_numpy(ops, grid.signals, grid.t_start, grid.t_end, 40, psi0)
    assert rel_fro(got, want) <= 1e-12
