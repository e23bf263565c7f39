"""The int8 tensor-core path (tcgen05 kind::i8, TMEM accumulators, TMA):
the int8 GEMM is exact (int32) against an integer reference; one Ozaki-sliced
real product is at FP64 level with 8 slices (and degrades by 2^-7 per slice
removed, as the scheme predicts); the Hermitian expm on both engines agrees
with the oracle."""
import ctypes

import numpy as np
import pytest

from conftest import rel_fro
from oracle import expm_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    from paper_2411_09982_b200 import _lib

    return _lib


@pytest.mark.parametrize("m,n,k", [(128, 128, 128), (200, 136, 160), (256, 384, 512), (1024, 512, 4096)])
def test_i8gemm_exact(L, m, n, k):
    import torch

    g = torch.Generator().manual_seed(m + n + k)
    a = torch.randint(-127, 128, (m, k), generator=g, dtype=torch.int8)
    b = torch.randint(-127, 128, (n, k), generator=g, dtype=torch.int8)
    da, db = a.cuda(), b.cuda()
    dc = torch.zeros(m, n, dtype=torch.int32, device="cuda")
    L.call("qch_i8gemm_test", L.dptr(da), L.dptr(db), L.dptr(dc), m, n, k, L.stream_ptr())
    ref = (a.long().double() @ b.long().double().T).round().long()
    assert torch.equal(dc.cpu().long(), ref)


@pytest.mark.parametrize("comp,k", [((0, 0), 1024), ((1, 4), 1024), ((2, 3), 1024), ((0, 1), 1001)])
def test_ozaki_real_product_accuracy(L, comp, k):
    import torch

    rng = np.random.default_rng(7)
    m, n = 384, 256
    x = rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k))
    y = rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k))
    x[5] *= 1e-7  # rows of very different scale keep their own exponent
    f = {0: lambda z: z.real, 1: lambda z: z.imag, 2: lambda z: z.real + z.imag, 3: lambda z: z.real - z.imag,
         4: lambda z: -z.imag}
    ref = f[comp[0]](x) @ f[comp[1]](y).T
    dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    errs = {}
    for s in (6, 8):
        out = torch.zeros(m, n, dtype=torch.float64, device="cuda")
        L.call("qch_oz_real_test", L.dptr(dx), comp[0], L.dptr(dy), comp[1], L.dptr(out), m, n, k, s, L.stream_ptr())
        got = out.cpu().numpy()
        scale = np.abs(f[comp[0]](x)).max(axis=1)[:, None] * np.abs(f[comp[1]](y)).max(axis=1)[None, :] * k
        errs[s] = float((np.abs(got - ref) / scale).max())
    assert errs[8] <= 1e-16          # FP64 level relative to the row/column scale
    assert errs[6] > 100 * errs[8]   # two slices less: ~2^-14 worse


@pytest.mark.parametrize("n", [512, 640, 601])
def test_expm_both_engines_vs_oracle(L, n):
    import paper_2411_09982_b200 as E

    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    h = (a + a.conj().T) * (0.3 / np.sqrt(n))
    ref = expm_oracle.expm_minus_i(h)
    old = L.load().qch_set_herm_gemm(-1)
    try:
        for engine in (1, 0):
            L.load().qch_set_herm_gemm(engine)
            assert rel_fro(E.expm_unitary(h).entries, ref) <= 1e-12, engine
    finally:
        L.load().qch_set_herm_gemm(old)


@pytest.mark.parametrize("n,batch", [(512, 1), (528, 3), (517, 2)])
def test_herm_products_int8_vs_fp64(L, n, batch):
    """qch_zgemm_herm_batched on the int8 engine: A A (one slicing for both
    sides) and A p(A) (distinct operands) for a batch, against numpy, with the
    lower-triangle result mirrored exactly (off-diagonal C Hermitian bit for bit)."""
    import torch

    rng = np.random.default_rng(n + batch)
    a = rng.standard_normal((batch, n, n)) + 1j * rng.standard_normal((batch, n, n))
    a = (a + np.conj(np.swapaxes(a, 1, 2))) / np.sqrt(n)
    p = a @ a * 0.5 - 0.25 * a  # a polynomial of a: commutes with a, A p Hermitian
    p = (p + np.conj(np.swapaxes(p, 1, 2))) / 2
    ddev = lambda z: torch.from_numpy(np.ascontiguousarray(z)).cuda()
    old = L.load().qch_set_herm_gemm(1)
    try:
        for x, y in ((a, a), (a, p)):
            dx = ddev(x)
            dy = dx if y is x else ddev(y)
            dc = torch.zeros_like(dx)
            L.call("qch_zgemm_herm_batched", L.dptr(dx), L.dptr(dy), L.dptr(dc), n, batch, L.stream_ptr())
            got = dc.cpu().numpy()
            ref = x @ y
            assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
            off = ~np.eye(n, dtype=bool)
            np.testing.assert_array_equal(got[:, off], np.conj(np.swapaxes(got, 1, 2))[:, off])
    finally:
        L.load().qch_set_herm_gemm(old)


def test_nonfinite_operator_takes_dmma_and_propagates_nan(L):
    """A NaN in an N > 4 operator reaching the propagator stage: the int8
    slices cannot carry it, so that batch runs on the DMMA products, which
    propagate the NaN as numpy's expm would — the trajectory must not come
    back finite (an error, or NaN states, as the reference)."""
    import paper_2411_09982_b200 as E

    ch = E.heisenberg_chain_hamiltonians(9)  # dim 512: the int8 engine's range
    d = ch.drift.to_dense().copy()
    d[3, 3] = np.nan
    ch2 = E.ControlledHamiltonian(E.HermitianOperator(d, validate=False), ch.controls)
    pulse = E.synthetic_transfer_pulse(1.0, 2 * 8 + 1, seed=1)
    grid = E.ControlGrid(0.0, 1.0, pulse.signals)
    psi0 = np.zeros(512, dtype=complex)
    psi0[0] = 1
    try:
        traj = E.evolve(ch2, grid, 2, psi0, order=2, check=False)
    except (E.NonFinite, E.NormDrift):
        return
    assert np.isnan(np.asarray(traj.amplitudes)[1:]).any()


@pytest.mark.parametrize("scale", [1e-6, 1e-3, 0.05, 0.45, 3.0])
def test_adaptive_slice_plan_matches_full_slices(L, scale, monkeypatch):
    """The adaptive plan (fewer slices for the products that reach U through
    small coefficients / high powers) against every product on 8 slices and
    against the oracle, over norms below, near and above the scaling target."""
    import paper_2411_09982_b200 as E

    n = 640
    rng = np.random.default_rng(int(scale * 100))
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    h = (a + a.conj().T)
    h *= scale / np.abs(h).sum(axis=1).max()  # ||H||_inf = scale
    monkeypatch.setenv("QCH_OZ_ADAPT", "0")
    full = E.expm_unitary(h).entries
    monkeypatch.setenv("QCH_OZ_ADAPT", "1")
    adapt = E.expm_unitary(h).entries
    assert rel_fro(adapt, full) <= 1e-15
    assert rel_fro(adapt, expm_oracle.expm_minus_i(h)) <= 1e-12


def test_int8_expm_rows_of_disparate_scale(L):
    """Per-row exponents: a Hermitian operator whose rows span 12 orders of
    magnitude (a diagonal similarity of a random Hermitian keeps it
    Hermitian only for real scalings, so use a block-diagonal mix) — the
    int8 engine against the DMMA engine and the oracle."""
    import paper_2411_09982_b200 as E

    n = 576
    rng = np.random.default_rng(11)
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    h = (a + a.conj().T) / np.sqrt(n)
    d = np.logspace(-12, 0, n)
    h = h * np.sqrt(np.outer(d, d))  # Hermitian, row/column scales from 1e-12 to 1
    h *= 0.4 / np.abs(h).sum(axis=1).max()
    old = L.load().qch_set_herm_gemm(-1)
    try:
        L.load().qch_set_herm_gemm(1)
        u8 = E.expm_unitary(h).entries
        L.load().qch_set_herm_gemm(0)
        ud = E.expm_unitary(h).entries
    finally:
        L.load().qch_set_herm_gemm(old)
    ref = expm_oracle.expm_minus_i(h)
    assert rel_fro(u8, ref) <= 1e-13
    assert rel_fro(u8, ud) <= 1e-13
