"""The Ozaki digit cut on the FP64 pipe (QCH_OZ_FPCUT=1, default) against
the 64-bit integer-shift form (QCH_OZ_FPCUT=0): one int8 Ozaki real product
(qch_oz_real_test) on rows spanning the whole double range — tiny rows that
take the integer fallback, subnormal entries, zeros, negative values — and an
exp(-iH) batch on the int8 engine must be identical BIT FOR BIT.  Each mode
runs in a child process (the switch is read once per process)."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

CHILD = r"""
import sys, ctypes, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2411_09982_b200 import _lib
L = _lib.load()
rng = np.random.default_rng(5)
m, n, k = 96, 64, 300
x = rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k))
y = rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k))
x *= np.exp2(rng.integers(-1000, 1000, size=(m, 1)).astype(float))
x[0] *= 1e-20                     # a row near the bottom of the range
x[1, :] = 5e-324 * rng.integers(-9, 9, size=k)  # subnormal entries only
x[2, ::3] = 0.0
y[3] *= 2.0 ** -1020
out = []
for s in (8, 5, 3):
    for comp in (0, 1, 2, 3):
        dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        o = torch.zeros((m, n), dtype=torch.float64, device="cuda")
        assert L.qch_oz_real_test(_lib.dptr(dx), comp, _lib.dptr(dy), comp, _lib.dptr(o), m, n, k, s,
                                  _lib.stream_ptr()) == 0, _lib.last_error()
        out.append(o.cpu().numpy())
nn, b = 512, 2
a = rng.standard_normal((b, nn, nn)) + 1j * rng.standard_normal((b, nn, nn))
h = (a + np.conj(np.transpose(a, (0, 2, 1)))) * (0.6 / np.sqrt(nn))
h[1] *= 1e-3
d_h = torch.from_numpy(h).cuda()
u = torch.empty_like(d_h)
work = torch.empty((8 * b, nn, nn), dtype=torch.complex128, device="cuda")
bad = ctypes.c_int64(-1)
assert L.qch_expm_minus_i_batch_c128(_lib.dptr(d_h), b, nn, _lib.dptr(u), _lib.dptr(work), ctypes.byref(bad),
                                     _lib.stream_ptr()) == 0, _lib.last_error()
out.append(np.ascontiguousarray(torch.view_as_real(u.cpu())).reshape(-1))
np.savez(sys.argv[2], *out)
"""


def test_fp_cut_bitwise_equals_integer_cut(tmp_path):
    res = []
    for mode in ("0", "1"):
        f = tmp_path / f"r{mode}.npz"
        env = dict(os.environ, QCH_OZ_FPCUT=mode)
        subprocess.run([sys.executable, "-c", CHILD, str(ROOT), str(f)], check=True, env=env, timeout=600)
        res.append(np.load(f))
    a, b = res
    assert list(a.keys()) == list(b.keys())
    for key in a.keys():
        assert np.array_equal(a[key].view(np.uint64), b[key].view(np.uint64)), key
