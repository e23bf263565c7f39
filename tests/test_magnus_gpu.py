"""Magnus / expm on the GPU vs the oracle and the reference's golden vectors.
Bar: 1e-10 relative (Frobenius) on matrices and trajectories."""
import numpy as np
import pytest

from conftest import rel_fro
from oracle import expm_oracle, magnus_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    import paper_2411_09982_b200 as eff

    return eff


def _ch(E, drift, controls):
    return E.ControlledHamiltonian(E.HermitianOperator(drift), [E.HermitianOperator(c) for c in controls])


def test_expm_vs_reference_golden(E, golden):
    g = golden("expm")
    for key in [k for k in g if k.startswith("h")]:
        u = E.expm_unitary(g[key]).entries
        assert rel_fro(u, g["u" + key[1:]]) <= 1e-12, key


def test_expm_batch_and_validate(E):
    rng = np.random.default_rng(0)
    hs = []
    for n in (3, 3, 3, 17, 17):
        a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        hs.append((a + a.conj().T) * 0.8)
    props = E.expm_batch(hs)
    for h, p in zip(hs, props):
        assert rel_fro(p.entries, expm_oracle.expm_minus_i(h)) <= 1e-12
        assert p.unitarity_defect() <= 1e-12
    bad = np.full((3, 3), np.nan)
    with pytest.raises(E.NonFinite):
        E.expm_batch([hs[0], bad])
    with pytest.raises(E.NonFinite):
        E.UnitaryPropagator(2 * np.eye(3, dtype=complex)).validate()


@pytest.mark.parametrize("n", [17, 100, 300])
def test_validate_determinant_branch(E, n):
    # expm.py:40-47 checks ||UU^dag - I||_F <= 1e-10 N AND ||det U| - 1| <= 1e-8.
    # The device evaluates |det U| from tr(UU^dag) and ||UU^dag - I||_F (no
    # LU); the decisions must equal numpy's on both sides of each bound.
    rng = np.random.default_rng(n)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    for eps in (0.0, 2e-12, 3e-10, 2e-9):
        u = (1.0 + eps) * q
        defect_ok = np.linalg.norm(u @ u.conj().T - np.eye(n)) <= 1e-10 * n
        det_ok = abs(abs(np.linalg.det(u)) - 1.0) <= 1e-8
        if defect_ok and det_ok:
            E.UnitaryPropagator(u).validate()
        else:
            with pytest.raises(E.NonFinite):
                E.UnitaryPropagator(u).validate()
    if n >= 100:  # scale passes the defect bound but not the determinant bound
        u = (1.0 + 3e-10) * q
        assert np.linalg.norm(u @ u.conj().T - np.eye(n)) <= 1e-10 * n
        assert abs(abs(np.linalg.det(u)) - 1.0) > 1e-8


@pytest.mark.parametrize("case", ["magnus_transmon_m2000", "magnus_spin6_m20"])
def test_evolve_order1_vs_reference_golden(E, golden, case):
    g = golden(case)
    t0, t1 = g["t"]
    m = int(g["m"])
    ch = _ch(E, g["drift"], g["controls"])
    grid = E.ControlGrid(t0, t1, g["signals"])
    np.testing.assert_array_equal(E.magnus_coefficients(grid, m), g["coeffs"])
    traj = E.evolve(ch, grid, m, g["psi0"])
    assert rel_fro(traj.amplitudes, g["traj"]) <= 1e-10
    if "hbar_head" in g:
        iv = E.magnus_intervals(ch, grid, m)
        hb = np.stack([iv.effective_hams[k].data for k in range(16)])
        assert rel_fro(hb, g["hbar_head"]) <= 1e-14
        _, props = E.evolve(ch, grid, m, g["psi0"], return_propagators=True)
        assert rel_fro(np.stack([p.entries for p in props[:16]]), g["u_head"]) <= 1e-12


@pytest.mark.parametrize("m", [1, 7, 300, 1000])
def test_evolve_order2_transmon_vs_oracle(E, m):
    ch, grid = E.driven_transmon(3, intervals=m, sub=4)
    d0 = ch.drift.data
    ctr = np.stack([c.data for c in ch.controls])
    psi0 = np.array([1, 0, 0], dtype=complex)
    ref = magnus_oracle.evolve(d0, ctr, grid.signals, grid.t_start, grid.t_end, m, psi0, order=2)
    got = E.evolve(ch, grid, m, psi0, order=2)
    assert rel_fro(got.amplitudes, ref) <= 1e-10
    c2 = E.magnus_coefficients_second_order(grid, m)
    np.testing.assert_array_equal(c2, magnus_oracle.second_order_coefficients(grid.signals, grid.t_start, grid.t_end, m))


def test_evolve_order2_spin_chain_vs_oracle(E, golden):
    g = golden("magnus_spin6_m20")
    t0, t1 = g["t"]
    ch = _ch(E, g["drift"], g["controls"])
    grid = E.ControlGrid(t0, t1, g["signals"])
    ref = magnus_oracle.evolve(g["drift"], g["controls"], g["signals"], t0, t1, 20, g["psi0"], order=2)
    got = E.evolve(ch, grid, 20, g["psi0"], order=2)
    assert rel_fro(got.amplitudes, ref) <= 1e-10
    iv = E.magnus_intervals(ch, grid, 20, order=2)
    hb = magnus_oracle.effective_hamiltonians(g["drift"], g["controls"], g["signals"], t0, t1, 20, order=2)
    assert rel_fro(iv.effective_hams.to_numpy(), hb) <= 1e-13


def test_evolve_large_dim_heisenberg_vs_oracle(E):
    # dim 256 (L = 8) exercises the DMMA Taylor path and the chain kernel
    ch = E.heisenberg_chain_hamiltonians(8)
    grid = E.synthetic_transfer_pulse(2.0, 4 * 8 + 1, seed=7)
    psi0 = np.zeros(256, dtype=complex)
    psi0[0] = 1
    d0 = ch.drift.to_dense()
    ctr = np.stack([c.to_dense() for c in ch.controls])
    for order in (1, 2):
        ref = magnus_oracle.evolve(d0, ctr, grid.signals, grid.t_start, grid.t_end, 4, psi0, order=order)
        got = E.evolve(ch, grid, 4, psi0, order=order)
        assert rel_fro(got.amplitudes, ref) <= 1e-10


def test_constant_hamiltonian_exactness(E):
    # SPEC AC5: time-independent evolution == eigendecomposition, any M
    rng = np.random.default_rng(1)
    a = rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))
    h = (a + a.conj().T) / 2
    ch = E.ControlledHamiltonian(E.HermitianOperator(h))
    psi0 = np.array([1, 0, 0, 0], dtype=complex)
    w, v = np.linalg.eigh(h)
    exact = v @ (np.exp(-1j * w * 2.0) * (v.conj().T @ psi0))
    for m in (1, 10, 100):
        grid = E.ControlGrid(0.0, 2.0, samples=m + 1)
        traj = E.evolve(ch, grid, m, psi0)
        assert np.linalg.norm(traj.amplitudes[-1] - exact) <= 1e-10


def test_magnus_errors(E):
    ch, grid = E.driven_transmon(3, intervals=10, sub=4)
    with pytest.raises(E.GridMismatch):
        E.magnus_coefficients(grid, 7)
    with pytest.raises(E.GridMismatch):
        E.evolve(ch, grid, 0, np.array([1, 0, 0], dtype=complex))
    with pytest.raises(E.DimensionMismatch):
        E.evolve(ch, grid, 10, np.array([1, 0], dtype=complex))
    with pytest.raises(ValueError):
        E.evolve(ch, grid, 10, np.array([1, 1, 0], dtype=complex))
    with pytest.raises(E.DimensionMismatch):
        E.assemble_effective_hams(ch, np.zeros((10, 3)), 0.1)


def test_zgemm_dmma_vs_numpy(E):
    import torch
    from paper_2411_09982_b200 import _lib

    rng = np.random.default_rng(3)
    for m, n, k, b in [(64, 64, 64, 1), (100, 37, 129, 3), (1, 1, 1, 2), (257, 130, 65, 1), (128, 64, 8, 2),
                       (300, 200, 77, 2), (513, 511, 1030, 1)]:
        a = rng.standard_normal((b, m, k)) + 1j * rng.standard_normal((b, m, k))
        bb = rng.standard_normal((b, k, n)) + 1j * rng.standard_normal((b, k, n))
        da, db = _lib.to_device(a), _lib.to_device(bb)
        dc = torch.empty((b, m, n), dtype=torch.complex128, device="cuda")
        _lib.call("qch_zgemm_batched", _lib.dptr(da), _lib.dptr(db), _lib.dptr(dc), m, n, k, b, m * k, k * n, m * n,
                  _lib.stream_ptr())
        assert rel_fro(dc.cpu().numpy(), a @ bb) <= 1e-14


@pytest.mark.parametrize("n,k", [(3, 10), (6, 9)])
def test_many_controls_generic_path(E, n, k):
    # more than 8 controls: the fused kernel's limit; these take the generic
    # device path (coefficients one at a time, assembly without register
    # arrays) — reference semantics for any K
    rng = np.random.default_rng(10 * n + k)

    def herm(scale):
        a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        return (a + a.conj().T) * scale

    ch = E.ControlledHamiltonian(E.HermitianOperator(herm(0.5)), [E.HermitianOperator(herm(0.05)) for _ in range(k)])
    m, sub = 200, 3
    grid = E.ControlGrid(0.0, 10.0, np.cos(np.outer(np.arange(1, k + 1), np.linspace(0, 4, m * sub + 1))))
    psi0 = np.zeros(n, complex)
    psi0[0] = 1
    d0 = ch.drift.data
    ctr = np.stack([c.data for c in ch.controls])
    for order in (1, 2):
        ref = magnus_oracle.evolve(d0, ctr, grid.signals, grid.t_start, grid.t_end, m, psi0, order=order)
        got = E.evolve(ch, grid, m, psi0, order=order)
        assert rel_fro(got.amplitudes, ref) <= 1e-10
    np.testing.assert_array_equal(E.magnus_coefficients(grid, m),
                                  magnus_oracle.first_order_coefficients(grid.signals, grid.t_start, grid.t_end, m))


def test_config5_first_intervals_vs_reference_itself(E):
    # BASELINE config 5 (12-spin Heisenberg chain, dim 4096) through the DMMA
    # path: its first 2 intervals at order 1 against the reference's evolve
    from pathlib import Path

    g = np.load(Path(__file__).parent / "golden" / "magnus_config5_first2_ref.npz")
    ch = E.heisenberg_chain_hamiltonians(12)
    grid = E.ControlGrid(0.0, float(g["t_end"]), g["signals"])
    psi0 = np.zeros(4096, dtype=complex)
    psi0[0] = 1.0
    got = E.evolve(ch, grid, 2, psi0, order=1, check=True)
    assert rel_fro(got.amplitudes, g["traj"]) <= 1e-10


def _herm(rng, n, scale=1.0):
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    return (a + a.conj().T) * (0.5 * scale)


@pytest.mark.parametrize("n,b", [(64, 1), (100, 3), (129, 2), (300, 1), (5, 4)])
def test_zgemm_herm_vs_numpy(E, n, b):
    # product of two commuting Hermitian factors (H^2 and H^3 = H^2 H): only
    # the lower tiles are computed, the upper triangle is the exact mirror
    import torch
    from paper_2411_09982_b200 import _lib

    rng = np.random.default_rng(n + b)
    h = np.stack([_herm(rng, n) for _ in range(b)])
    h2 = h @ h
    dh, dh2 = _lib.to_device(h), _lib.to_device(h2)
    out = torch.empty((b, n, n), dtype=torch.complex128, device="cuda")
    _lib.call("qch_zgemm_herm_batched", _lib.dptr(dh2), _lib.dptr(dh), _lib.dptr(out), n, b, _lib.stream_ptr())
    got = out.cpu().numpy()
    assert rel_fro(got, h2 @ h) <= 1e-14
    iu = np.triu_indices(n, 1)
    for q in range(b):
        np.testing.assert_array_equal(got[q][iu], got[q].T[iu].conj())


@pytest.mark.parametrize("n", [100, 300])
def test_unitarity_defect_vs_numpy(E, n):
    import torch
    from paper_2411_09982_b200 import _lib

    rng = np.random.default_rng(n)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    u = q * (1.0 + 1e-6 * rng.standard_normal(n))
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    _lib.call("qch_unitarity_defect_c128", _lib.dptr(_lib.to_device(u)), 1, n, _lib.dptr(out), _lib.stream_ptr())
    want = np.linalg.norm(u @ u.conj().T - np.eye(n))
    assert abs(float(out.item()) - want) <= 1e-9 * want


@pytest.mark.parametrize("n,scale", [(17, 0.3), (64, 0.05), (130, 1.0), (256, 8.0)])
def test_expm_hermitian_and_general_paths_vs_oracle(E, n, scale):
    # bitwise-Hermitian input -> cos/sin form on Hermitian half-GEMMs; the
    # same matrix with a 1e-9 non-Hermitian part -> the general
    # Paterson-Stockmeyer path; both against the reference's 18-term Taylor
    rng = np.random.default_rng(7 * n)
    h = _herm(rng, n, scale)
    assert np.array_equal(h, h.conj().T)
    assert rel_fro(E.expm_unitary(h).entries, expm_oracle.expm_minus_i(h)) <= 1e-12
    g = h + 1e-9 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    assert rel_fro(E.expm_unitary(g, check=False).entries, expm_oracle.expm_minus_i(g)) <= 1e-12
    hs = [_herm(rng, n, scale) for _ in range(3)]
    for h_, p in zip(hs, E.expm_batch(hs)):
        assert rel_fro(p.entries, expm_oracle.expm_minus_i(h_)) <= 1e-12


def test_config5_order2_vs_oracle(E):
    # BASELINE config 5 at ORDER 2 (the configured order; the reference has
    # no second order): the first 3 of its 4096 intervals against the oracle
    # (magnus_oracle.evolve, 18-term Taylor as expm.py:56-71; made by
    # oracle/gen_golden_long.py), through the device path with check=True
    from pathlib import Path

    g = np.load(Path(__file__).parent / "golden" / "magnus_config5_order2_oracle.npz")
    ch = E.heisenberg_chain_hamiltonians(12)
    grid = E.ControlGrid(0.0, float(g["t_end"]), g["signals"])
    psi0 = np.zeros(4096, dtype=complex)
    psi0[0] = 1.0
    got = E.evolve(ch, grid, 3, psi0, order=2, check=True)
    assert rel_fro(got.amplitudes, g["traj"]) <= 1e-10
    # mid-pulse intervals (2048, 2049), where the second-order term is large
    # (the pulse starts near zero)
    gm = np.load(Path(__file__).parent / "golden" / "magnus_config5_mid_order2_oracle.npz")
    t0, t1 = (float(x) for x in gm["t"])
    gridm = E.ControlGrid(t0, t1, gm["signals"])
    psim = gm["traj"][0]
    got2 = E.evolve(ch, gridm, 2, psim, order=2, check=True)
    assert rel_fro(got2.amplitudes, gm["traj"]) <= 1e-10
    got1 = E.evolve(ch, gridm, 2, psim, order=1, check=False)
    # the second-order term is small at this grid spacing (dt = 25/4096) but
    # well above the tolerance: order 1 misses the golden by ~4e-9
    assert rel_fro(got1.amplitudes, gm["traj"]) > 10 * 1e-10


@pytest.mark.parametrize("order", [1, 2])
def test_return_propagators_large_dim_vs_oracle(E, order):
    # N = 64 (DMMA path): evolve(..., return_propagators=True) returns the
    # reference's list of UnitaryPropagator (magnus.py:262-266), each equal to
    # the oracle's exp(-i Hbar_n); check=True validates every one
    ch = E.heisenberg_chain_hamiltonians(6)
    grid = E.synthetic_transfer_pulse(3.0, 12 * 4 + 1, seed=11)
    psi0 = np.zeros(64, dtype=complex)
    psi0[0] = 1
    traj, props = E.evolve(ch, grid, 12, psi0, order=order, check=True, return_propagators=True)
    d0 = ch.drift.to_dense()
    ctr = np.stack([c.to_dense() for c in ch.controls])
    ref_traj, ref_u = magnus_oracle.evolve(d0, ctr, grid.signals, grid.t_start, grid.t_end, 12, psi0, order=order,
                                           return_propagators=True)
    assert len(props) == 12 and all(isinstance(p, E.UnitaryPropagator) for p in props)
    assert rel_fro(np.stack([p.entries for p in props]), ref_u) <= 1e-12
    assert rel_fro(traj.amplitudes, ref_traj) <= 1e-10
    assert np.array_equal(traj.times, np.linspace(grid.t_start, grid.t_end, 13))


@pytest.mark.parametrize("n,scale,b", [(512, 0.2, 2), (1024, 0.05, 1), (768, 3.0, 1)])
def test_expm_hermitian_int8_tensor_path_vs_oracle(E, n, scale, b):
    # n >= 512: the Hermitian products run on the int8 tensor cores (Ozaki
    # slices, tcgen05; ozgemm.cu) — same 1e-12 bar as the DMMA path against
    # the reference's 18-term Taylor (scale 3: squarings on the DMMA path)
    rng = np.random.default_rng(n)
    hs = [_herm(rng, n, scale / np.sqrt(n)) for _ in range(b)]
    for h, p in zip(hs, E.expm_batch(hs)):
        assert rel_fro(p.entries, expm_oracle.expm_minus_i(h)) <= 1e-12


@pytest.mark.parametrize("n", [512, 1000, 1024])
def test_zgemm_herm_int8_tensor_path_vs_numpy(E, n):
    import torch
    from paper_2411_09982_b200 import _lib

    rng = np.random.default_rng(n + 1)
    h = _herm(rng, n)
    h2 = h @ h
    out = torch.empty((1, n, n), dtype=torch.complex128, device="cuda")
    dh2, dh = _lib.to_device(h2), _lib.to_device(h)  # (kept alive across the call)
    _lib.call("qch_zgemm_herm_batched", _lib.dptr(dh2), _lib.dptr(dh), _lib.dptr(out), n, 1, _lib.stream_ptr())
    got = out[0].cpu().numpy()
    assert rel_fro(got, h2 @ h) <= 1e-14
    iu = np.triu_indices(n, 1)
    np.testing.assert_array_equal(got[iu], got.T[iu].conj())


@pytest.mark.parametrize("pos", [(5, 5), (70, 3), (99, 98), (40, 64)])
def test_expm_nearly_hermitian_takes_general_path(E, pos):
    # Hermitian except ONE entry (an imaginary diagonal entry, or one
    # off-diagonal entry in a diagonal / off-diagonal / last partial tile):
    # the Hermitian-only (half-GEMM) path must not be taken
    from oracle import expm_oracle

    n = 100
    rng = np.random.default_rng(sum(pos))
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    h = (a + a.conj().T) * (0.3 / np.sqrt(n))
    r, c = pos
    h[r, c] += 0.05j if r == c else 0.05
    got = E.expm_batch([h], check=False)[0].entries
    ref = expm_oracle.expm_minus_i(h)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-10
