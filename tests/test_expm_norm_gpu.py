"""The scaling norm of _expm_minus_i (expm.py:59: max over rows of
np.abs(-1j * h).sum(axis=1)) on the device, qch_expm_norm_c128, equals
numpy's value BIT FOR BIT (it picks the number of squarings, expm.py:61-63)
for every leaf shape of numpy's pairwise tree: n < 8, 8..128 with a
remainder, and split trees above 128 (ragged n included)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 5, 7, 8, 9, 17, 64, 100, 127, 128, 129, 200, 256, 300, 513, 1000, 2049])
def test_norm_bitwise_numpy(n):
    import torch

    from paper_2411_09982_b200 import _lib

    batch = 3 if n <= 1000 else 1
    rng = np.random.default_rng(n)
    h = rng.standard_normal((batch, n, n)) + 1j * rng.standard_normal((batch, n, n))
    h *= np.exp(rng.uniform(-20, 20, size=(batch, n, 1)))  # rows over many binades
    h[:, 0, :] = 0.0
    want = np.array([float(np.max(np.abs(-1j * x).sum(axis=1))) for x in h])
    d_h = torch.from_numpy(h).cuda()
    out = torch.empty(batch, dtype=torch.float64, device="cuda")
    assert _lib.load().qch_expm_norm_c128(_lib.dptr(d_h), batch, n, _lib.dptr(out), _lib.stream_ptr()) == 0
    got = out.cpu().numpy()
    np.testing.assert_array_equal(got, want)
