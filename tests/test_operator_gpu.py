"""HermitianOperator validation for large dense host matrices runs on the
device (qch_hermitian_defect_c128 + the max_abs kernel): same values and the
same decisions as the reference's numpy scan (operators.py:92-116)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    import paper_2411_09982_b200 as eff

    return eff


@pytest.mark.parametrize("n", [512, 777, 1024])
def test_device_validation_matches_numpy(E, n):
    from paper_2411_09982_b200 import operators

    assert n >= operators.DEVICE_CHECK_DIM
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    h = (a + a.conj().T) / 2
    op = E.HermitianOperator(h)  # bitwise Hermitian: passes
    assert op.max_abs() == float(np.max(np.abs(h)))
    scale = float(np.max(np.abs(h)))
    for rel, ok in ((5e-13, True), (2e-12, False)):
        g = h.copy()
        g[n // 3, n // 5] += rel * scale
        worst = float(np.max(np.abs(g - g.conj().T)))
        assert (worst <= 1e-12 * scale) == ok
        if ok:
            E.HermitianOperator(g)
        else:
            with pytest.raises(E.HermiticityViolation):
                E.HermitianOperator(g)


def test_exact_hermitian_flag_tiles(E):
    import torch

    from paper_2411_09982_b200 import _lib

    for n in (1, 31, 33, 100, 257):
        rng = np.random.default_rng(n)
        a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        h = (a + a.conj().T) / 2
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.call("qch_hermitian_exact_c128", _lib.dptr(_lib.to_device(h)), n, _lib.dptr(flag), _lib.stream_ptr())
        assert int(flag.item()) == 0
        if n > 1:
            h[n - 1, 0] = complex(np.nextafter(h[n - 1, 0].real, np.inf), h[n - 1, 0].imag)  # one ulp
            _lib.call("qch_hermitian_exact_c128", _lib.dptr(_lib.to_device(h)), n, _lib.dptr(flag),
                      _lib.stream_ptr())
            assert int(flag.item()) == 1
