"""Device-side model builders: the spin chain of
models.py:288-325 built as device CSRs must equal the host builder (itself
the reference's statement) bit for bit — indptr, sorted indices, values —
and evolve to the same trajectory."""
import numpy as np
import pytest

from conftest import rel_fro

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    import paper_2411_09982_b200 as eff

    return eff


def _same(a, b):
    a, b = a.tocsr(), b.tocsr()
    np.testing.assert_array_equal(a.indptr, b.indptr)
    np.testing.assert_array_equal(a.indices, b.indices)
    np.testing.assert_array_equal(a.data, b.data)


@pytest.mark.parametrize("length", [3, 4, 5, 8, 11, 14])
@pytest.mark.parametrize("prm", [(0.3, 0.5, 0.2), (1.7, -0.31, 0.045), (0.0, 1.0, 0.0), (0.0, 0.0, 0.0)])
def test_spin_chain_device_builder_bit_exact(E, length, prm):
    # (0, 1, 0) and (0, 0, 0) leave exact zeros on the diagonal: dropped
    # from the CSR as scipy drops them
    p = E.SpinChainParams(length, *prm)
    host = E.spin_chain_hamiltonians(p)
    dev = E.spin_chain_hamiltonians_device(p)
    assert dev.dim == host.dim and dev.num_controls == 2
    _same(dev.drift.data, host.drift.data)
    for a, b in zip(dev.controls, host.controls):
        _same(a.data, b.data)
    assert dev.drift.max_abs() == host.drift.max_abs()


def test_spin_chain_device_builder_errors(E):
    from paper_2411_09982_b200.errors import ChainTooLarge

    with pytest.raises(ChainTooLarge):
        E.spin_chain_hamiltonians_device(E.SpinChainParams(15, 0.3, 0.5, 0.2))
    with pytest.raises(ValueError):
        E.SpinChainParams(2, 0.3, 0.5, 0.2)


def test_spin_chain_device_densify(E):
    # device_tensor of a device CSR scatters on the device, no host round trip
    p = E.SpinChainParams(6, 0.3, 0.5, 0.2)
    dev, host = E.spin_chain_hamiltonians_device(p), E.spin_chain_hamiltonians(p)
    for a, b in zip([dev.drift] + dev.controls, [host.drift] + host.controls):
        assert a._m is None
        np.testing.assert_array_equal(a.device_tensor().cpu().numpy(), b.data.toarray())


def test_spin_chain_device_evolve_matches_host(E):
    p = E.SpinChainParams(7, 0.3, 0.5, 0.2)
    grid = E.synthetic_transfer_pulse(5.0, 2049, 11)
    psi0 = np.zeros(1 << 7, dtype=complex)
    psi0[0] = 1
    a = E.evolve(E.spin_chain_hamiltonians_device(p), grid, 512, psi0, order=2).amplitudes
    b = E.evolve(E.spin_chain_hamiltonians(p), grid, 512, psi0, order=2).amplitudes
    assert rel_fro(a, b) <= 1e-13


@pytest.mark.parametrize("length", [1, 2, 3])
def test_spin_chain_c_abi_short_chains(E, length):
    # the C-ABI accepts 1 <= L <= 30 (SpinChainParams needs L >= 3): the
    # reference's numpy expressions (models.py:302-320) stated directly
    import ctypes

    import scipy.sparse as sps
    import torch

    from paper_2411_09982_b200 import _lib

    w, jn, g2 = 0.7, 0.4, -0.25
    n = 1 << length
    idx = np.arange(n, dtype=np.int64)
    z = 1 - 2 * ((idx[:, None] >> np.arange(length)) & 1)
    diag = 0.5 * w * z.sum(axis=1) - jn * (z * np.roll(z, -1, axis=1)).sum(axis=1) \
        - g2 * (z * np.roll(z, -2, axis=1)).sum(axis=1)
    want = sps.diags(diag.astype(np.complex128), format="csr")
    ip = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    ix = torch.empty(n, dtype=torch.int32, device="cuda")
    dv = torch.empty(n, dtype=torch.complex128, device="cuda")
    nnz = ctypes.c_int64(-1)
    _lib.call("qch_build_spin_chain_drift_c128", length, w, jn, g2, _lib.dptr(ip), _lib.dptr(ix), _lib.dptr(dv),
              ctypes.byref(nnz), _lib.stream_ptr())
    k = nnz.value
    got = sps.csr_matrix((dv[:k].cpu().numpy(), ix[:k].cpu().numpy(), ip.cpu().numpy()), shape=(n, n))
    _same(got, want)
    with pytest.raises(ValueError):
        _lib.call("qch_build_spin_chain_drift_c128", 31, w, jn, g2, _lib.dptr(ip), _lib.dptr(ix), _lib.dptr(dv),
                  ctypes.byref(nnz), _lib.stream_ptr())
