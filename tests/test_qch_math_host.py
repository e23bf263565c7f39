"""qch_math.cuh (the device numerics that reproduce numpy's rounding) compiled
for the HOST with g++ and compared bit-for-bit with numpy / math / the oracle."""
import ctypes
import math
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HARNESS = r'''
#include "qch_math.cuh"
extern "C" {
void cabs_v(const double* re, const double* im, double* out, int n) { for (int i = 0; i < n; ++i) out[i] = np_cabs(re[i], im[i]); }
void hypot_v(const double* x, const double* y, double* out, int n) { for (int i = 0; i < n; ++i) out[i] = hypot_cr(x[i], y[i]); }
void cmul_v(const double* a, const double* b, double* out, int n) {
  for (int i = 0; i < n; ++i) { cplx z = np_cmul(mkc(a[2*i], a[2*i+1]), mkc(b[2*i], b[2*i+1])); out[2*i] = z.re; out[2*i+1] = z.im; }
}
double pairwise(const double* a, int n) { auto f = [&](int k) { return a[k]; }; return np_pairwise(f, n); }
void block_v(double c, const double* s, const double* h4, double* out) {
  Block2 b = rotate_block(c, mkc(s[0], s[1]), mkc(h4[0], h4[1]), mkc(h4[2], h4[3]), mkc(h4[4], h4[5]), mkc(h4[6], h4[7]));
  double v[8] = {b.ii.re, b.ii.im, b.ij.re, b.ij.im, b.ji.re, b.ji.im, b.jj.re, b.jj.im};
  for (int k = 0; k < 8; ++k) out[k] = v[k];
}
}
'''


@pytest.fixture(scope="module")
def lib(tmp_path_factory):
    d = tmp_path_factory.mktemp("qchmath")
    src = d / "h.cpp"
    src.write_text(HARNESS)
    so = d / "h.so"
    subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-ffp-contract=off",
                    "-I", str(ROOT / "paper_2411_09982_b200" / "csrc"), "-I", "/usr/local/cuda/include",
                    str(src), "-o", str(so)], check=True)
    return ctypes.CDLL(str(so))


P = ctypes.POINTER(ctypes.c_double)


def _p(a):
    return a.ctypes.data_as(P)


def test_np_cabs_bitwise(lib):
    rng = np.random.default_rng(0)
    n = 100000
    re = rng.standard_normal(n) * np.exp(rng.uniform(-30, 30, n))
    im = rng.standard_normal(n) * np.exp(rng.uniform(-30, 30, n))
    re[:10] = 0.0
    out = np.empty(n)
    lib.cabs_v(_p(re), _p(im), _p(out), n)
    np.testing.assert_array_equal(out, np.abs(re + 1j * im))


def test_hypot_correctly_rounded(lib):
    rng = np.random.default_rng(1)
    n = 50000
    x = rng.standard_normal(n) * np.exp(rng.uniform(-20, 20, n))
    y = rng.standard_normal(n) * np.exp(rng.uniform(-20, 20, n))
    out = np.empty(n)
    lib.hypot_v(_p(x), _p(y), _p(out), n)
    np.testing.assert_array_equal(out, np.array([math.hypot(a, b) for a, b in zip(x, y)]))


def test_cmul_bitwise(lib):
    rng = np.random.default_rng(2)
    a = rng.standard_normal(20000) + 1j * rng.standard_normal(20000)
    b = rng.standard_normal(20000) + 1j * rng.standard_normal(20000)
    out = np.empty(40000)
    av, bv = a.view(np.float64).copy(), b.view(np.float64).copy()
    lib.cmul_v(_p(av), _p(bv), _p(out), 20000)
    np.testing.assert_array_equal(out.view(np.complex128), a * b)


@pytest.mark.parametrize("n", [1, 3, 4, 7, 8, 9, 15, 16, 100, 128, 129, 257, 1000, 4096])
def test_pairwise_sum_bitwise(lib, n):
    lib.pairwise.restype = ctypes.c_double
    rng = np.random.default_rng(n)
    a = rng.standard_normal(n) * np.exp(rng.uniform(-5, 5, n))
    assert lib.pairwise(_p(a), n) == a.reshape(1, n).sum(axis=1)[0]


def test_rotate_block_matches_oracle_rotation(lib):
    from oracle import npad_oracle

    rng = np.random.default_rng(3)
    for _ in range(300):
        a = rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2))
        h = (a + a.conj().T) / 2
        c, sh, ph, _ = npad_oracle.rotation_scalars(h, 0, 1)
        s = npad_oracle.block_s(sh, ph)
        ref = h.copy()
        npad_oracle.rotate(ref, 0, 1, c, s)
        out = np.empty(8)
        h4 = np.array([h[0, 0], h[0, 1], h[1, 0], h[1, 1]]).view(np.float64).copy()
        sv = np.array([s.real, s.imag])
        lib.block_v(ctypes.c_double(c), _p(sv), _p(h4), _p(out))
        got = out.view(np.complex128).reshape(2, 2)
        np.testing.assert_array_equal(got, ref)
