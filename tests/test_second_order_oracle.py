"""The second-order Magnus restatement (no reference implementation exists,
SPEC.md:14) checked against brute-force nested Gauss-Legendre quadrature of
X = int int_{t2<t1} [H(t1), H(t2)] for piecewise-linear controls, and its
accuracy gain over first order on the reference spin chain (SPEC AC7)."""
import numpy as np
import pytest

from oracle import expm_oracle, magnus_oracle


def _interp(sig, t, t_end):
    grid = np.linspace(0.0, t_end, sig.shape[1])
    return np.array([np.interp(t, grid, s) for s in sig])


def _brute_x(drift, controls, sig, t_end, order=24):
    """Nested Gauss-Legendre per sample panel (exact for piecewise-linear u)."""
    k = sig.shape[0]
    panels = sig.shape[1] - 1
    h = t_end / panels
    xg, wg = np.polynomial.legendre.leggauss(order)

    def ham(t):
        u = _interp(sig, t, t_end)
        return drift + sum(u[q] * controls[q] for q in range(k))

    x = np.zeros_like(drift)
    for a in range(panels):
        lo = a * h
        for xi, wi in zip(xg, wg):
            t1 = lo + (xi + 1) * h / 2
            h1 = ham(t1)
            # inner integral over [0, t1]: full panels + partial panel
            inner = np.zeros_like(drift)
            for b in range(a):
                for xj, wj in zip(xg, wg):
                    inner += wj * h / 2 * ham(b * h + (xj + 1) * h / 2)
            for xj, wj in zip(xg, wg):
                inner += wj * (t1 - lo) / 2 * ham(lo + (xj + 1) * (t1 - lo) / 2)
            x += wi * h / 2 * (h1 @ inner - inner @ h1)
    return x


@pytest.mark.parametrize("k,sub,seed", [(1, 3, 0), (2, 4, 1), (3, 2, 2)])
def test_second_order_closed_form_vs_quadrature(k, sub, seed):
    rng = np.random.default_rng(seed)
    n = 3
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    drift = (a + a.conj().T) / 2
    controls = []
    for _ in range(k):
        b = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        controls.append((b + b.conj().T) / 2)
    controls = np.array(controls)
    t_end = 0.7
    sig = rng.standard_normal((k, sub + 1))
    c2 = magnus_oracle.second_order_coefficients(sig, 0.0, t_end, 1)[0]
    comm = magnus_oracle.commutators(drift, controls)
    x = sum(w * c for w, c in zip(c2, comm))
    ref = _brute_x(drift, controls, sig, t_end)
    assert np.linalg.norm(x - ref) <= 1e-13 * max(1.0, np.linalg.norm(ref))


def test_second_order_improves_spin_chain_accuracy():
    # SPEC AC7 setting (L = 6 ZZ chain, band-limited pulse): order 2 beats order 1
    from paper_2411_09982_b200 import models

    p = models.SpinChainParams(length=6, qubit_freq=1.0, j_nn=0.25, g_nnn=0.05)
    ch = models.spin_chain_hamiltonians(p)
    d0 = ch.drift.to_dense()
    ctr = np.stack([c.to_dense() for c in ch.controls])
    m_fine, m = 1600, 40
    grid = models.synthetic_transfer_pulse(25.0, m_fine * 2 + 1, seed=3)
    psi0 = np.zeros(64, dtype=complex)
    psi0[0] = 1
    fine = magnus_oracle.evolve(d0, ctr, grid.signals, 0.0, 25.0, m_fine, psi0, order=2)[-1]
    e1 = np.linalg.norm(magnus_oracle.evolve(d0, ctr, grid.signals, 0.0, 25.0, m, psi0, order=1)[-1] - fine)
    e2 = np.linalg.norm(magnus_oracle.evolve(d0, ctr, grid.signals, 0.0, 25.0, m, psi0, order=2)[-1] - fine)
    assert e2 < 0.2 * e1, (e1, e2)


def test_hbar2_is_hermitian():
    from paper_2411_09982_b200 import models

    ch, grid = models.driven_transmon(3, intervals=5, sub=4)
    hb = magnus_oracle.effective_hamiltonians(ch.drift.data, np.stack([c.data for c in ch.controls]), grid.signals,
                                              grid.t_start, grid.t_end, 5, order=2)
    for h in hb:
        assert np.linalg.norm(h - h.conj().T) <= 1e-14 * np.linalg.norm(h)
    u = expm_oracle.expm_minus_i(hb[2])
    assert expm_oracle.is_valid_propagator(u)
