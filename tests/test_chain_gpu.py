"""The ordered product psi <- U_m psi (magnus.py:249-252) through
qch_magnus_chain_c128 at both kernels' size ranges: the one-cluster DSMEM
chain (4 < N <= 384) and the cooperative grid (larger N; 4 rows per warp
above 1024), including ragged N and chunks of 1..3 intervals, against a
numpy sequential product (fp64, bar 1e-12 relative per row); and the
NormDrift check (magnus.py:270-273) flagging the first non-unitary interval
with its index."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _unitaries(n, m, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, n, n)) + 1j * rng.standard_normal((m, n, n))
    q, r = np.linalg.qr(a)
    d = np.diagonal(r, axis1=1, axis2=2)
    return q * (d / np.abs(d))[:, None, :]


def _chain(us, psi):
    import torch

    from paper_2411_09982_b200 import sharding

    comp = sharding.DeviceRelayCompute()
    d_u = torch.from_numpy(np.ascontiguousarray(us)).cuda()
    rows, err = comp.chain(d_u, us.shape[0], comp.to_tensor(psi))
    return rows.cpu().numpy(), err


def _ref(us, psi):
    out, x = [], psi
    for u in us:
        x = u @ x
        out.append(x)
    return np.stack(out)


@pytest.mark.parametrize("n,m", [(5, 9), (8, 3), (17, 30), (48, 5), (64, 64), (65, 7), (100, 3), (128, 40),
                                 (129, 2), (200, 17), (256, 33), (256, 1), (300, 9), (384, 12), (385, 4),
                                 (512, 6), (1100, 3), (2048, 2)])
def test_chain_vs_numpy(n, m):
    us = _unitaries(n, m, seed=n + m)
    rng = np.random.default_rng(n)
    psi = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    psi /= np.linalg.norm(psi)
    got, err = _chain(us, psi)
    assert err is None, err
    ref = _ref(us, psi)
    e = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert e.max() <= 1e-12, (e.max(), int(e.argmax()))


@pytest.mark.parametrize("n", [6, 100, 256, 384, 600])
def test_chain_norm_drift_index(n):
    m = 11
    us = _unitaries(n, m, seed=3)
    us[6] *= 1.001
    us[9] *= 1.5
    psi = np.zeros(n, dtype=complex)
    psi[1] = 1.0
    _, err = _chain(us, psi)
    assert err is not None
    st, bad, msg = err
    assert st == 9 and bad == 6, (st, bad, msg)
