// qch_math.cuh — scalar arithmetic that reproduces the reference's numpy/libm
// rounding on the device (and on the host, so the CPU tests can exercise it).
//
// Every helper here is pinned to a concrete operation of the reference:
//   np_cabs     numpy SIMD |z| used by np.abs(complex128) in selection and
//               max_abs (operators.py:98, npad.py:313): L*sqrt(fma(S/L,S/L,1))
//   np_cmul     numpy complex multiply, re = fma(ar,br,-(ai*bi)),
//               im = fma(ar,bi,ai*br) (npad.py:136-144, magnus.py:186-188)
//   hypot_cr    correctly rounded hypot (math.hypot, npad.py:117; glibc hypot
//               behind abs(complex), npad.py:114)
//   np_pairwise numpy's pairwise summation used by .sum(axis=...) (n<8
//               sequential; 8-accumulator blocks up to 128; recursive above),
//               magnus.py:166, expm.py:59
// Explicit __dmul_rn/__dadd_rn/__fma_rn stop nvcc from contracting a*b+c
// differently from numpy.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#define QCH_HD __host__ __device__ __forceinline__

#ifdef __CUDA_ARCH__
#define QMUL(a, b) __dmul_rn((a), (b))
#define QADD(a, b) __dadd_rn((a), (b))
#define QSUB(a, b) __dsub_rn((a), (b))
#define QFMA(a, b, c) __fma_rn((a), (b), (c))
#define QDIV(a, b) __ddiv_rn((a), (b))
#define QSQRT(a) __dsqrt_rn(a)
#else
#define QMUL(a, b) ((a) * (b))
#define QADD(a, b) ((a) + (b))
#define QSUB(a, b) ((a) - (b))
#define QFMA(a, b, c) fma((a), (b), (c))
#define QDIV(a, b) ((a) / (b))
#define QSQRT(a) sqrt(a)
#endif

struct cplx {
  double re, im;
};

QCH_HD cplx mkc(double r, double i) {
  cplx z;
  z.re = r;
  z.im = i;
  return z;
}
QCH_HD cplx d2c(double2 v) { return mkc(v.x, v.y); }
QCH_HD double2 c2d(cplx z) { return make_double2(z.re, z.im); }
QCH_HD cplx cconj(cplx a) { return mkc(a.re, -a.im); }
QCH_HD cplx cadd(cplx a, cplx b) { return mkc(QADD(a.re, b.re), QADD(a.im, b.im)); }
QCH_HD cplx csub(cplx a, cplx b) { return mkc(QSUB(a.re, b.re), QSUB(a.im, b.im)); }

// numpy complex128 multiply (AVX512F/AVX2 loops): FMA on the first product.
QCH_HD cplx np_cmul(cplx a, cplx b) {
  return mkc(QFMA(a.re, b.re, -QMUL(a.im, b.im)), QFMA(a.re, b.im, QMUL(a.im, b.re)));
}
// real scalar times complex: numpy promotes the scalar to (x + 0j) first.
QCH_HD cplx np_rmul(double x, cplx b) { return np_cmul(mkc(x, 0.0), b); }

// numpy complex division by a real-valued complex (k + 0j): Smith's algorithm
// with rat = 0 reduces to multiplication by the rounded reciprocal 1/k.
QCH_HD cplx np_cdiv_real(cplx a, double k) {
  double scl = QDIV(1.0, k);
  return mkc(QMUL(a.re, scl), QMUL(a.im, scl));
}

// numpy SIMD complex absolute value (loops_unary_complex: simd_cabsolute).
QCH_HD double np_cabs(double re, double im) {
  double a = fabs(re), b = fabs(im);
  if (isinf(a) || isinf(b)) return INFINITY;
  if (isnan(a) || isnan(b)) return NAN;
  double L = fmax(a, b), S = fmin(a, b);
  double r = (L == 0.0) ? 0.0 : QDIV(S, L);
  return QMUL(QSQRT(QFMA(r, r, 1.0)), L);
}
QCH_HD double np_cabs(cplx z) { return np_cabs(z.re, z.im); }

// Correctly rounded (in practice) hypot: Borges' fma-corrected algorithm with
// power-of-two prescaling.  Matches Python math.hypot / glibc hypot.
QCH_HD double hypot_cr(double x, double y) {
  x = fabs(x);
  y = fabs(y);
  if (isinf(x) || isinf(y)) return INFINITY;
  if (isnan(x) || isnan(y)) return NAN;
  if (x < y) {
    double t = x;
    x = y;
    y = t;
  }
  if (x == 0.0) return 0.0;
  // scale into a safe range by an exact power of two
  int e;
  frexp(x, &e);
  double sc = ldexp(1.0, -e);
  double xs = QMUL(x, sc), ys = QMUL(y, sc);  // xs in [0.5,1)
  // ys may underflow to subnormal when y << x; that only affects bits far below
  // the rounding position of the result.
  double h = QSQRT(QFMA(xs, xs, QMUL(ys, ys)));
  double h_sq = QMUL(h, h);
  double x_sq = QMUL(xs, xs);
  double dlt = QADD(QSUB(QFMA(-ys, ys, QSUB(h_sq, x_sq)), QFMA(xs, xs, -x_sq)), QFMA(h, h, -h_sq));
  h = QSUB(h, QDIV(dlt, QMUL(2.0, h)));
  return ldexp(h, e);
}

// numpy pairwise sum over a strided sequence produced by a functor f(idx).
// n < 8: sequential from 0.0; 8 <= n <= 128: 8 accumulators; larger: split.
template <typename F>
QCH_HD double np_pairwise_block(const F& f, int off, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = QADD(res, f(off + i));
    return res;
  }
  double r0 = f(off + 0), r1 = f(off + 1), r2 = f(off + 2), r3 = f(off + 3);
  double r4 = f(off + 4), r5 = f(off + 5), r6 = f(off + 6), r7 = f(off + 7);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
    r0 = QADD(r0, f(off + i + 0));
    r1 = QADD(r1, f(off + i + 1));
    r2 = QADD(r2, f(off + i + 2));
    r3 = QADD(r3, f(off + i + 3));
    r4 = QADD(r4, f(off + i + 4));
    r5 = QADD(r5, f(off + i + 5));
    r6 = QADD(r6, f(off + i + 6));
    r7 = QADD(r7, f(off + i + 7));
  }
  double res = QADD(QADD(QADD(r0, r1), QADD(r2, r3)), QADD(QADD(r4, r5), QADD(r6, r7)));
  for (; i < n; ++i) res = QADD(res, f(off + i));
  return res;
}

template <typename F>
#if defined(__CUDACC__)
#define QCH_NOINLINE __noinline__
#else
#define QCH_NOINLINE __attribute__((noinline))
#endif
__host__ __device__ QCH_NOINLINE double np_pairwise_rec(const F& f, int off, int n) {
  if (n <= 128) return np_pairwise_block(f, off, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return QADD(np_pairwise_rec(f, off, n2), np_pairwise_rec(f, off + n2, n - n2));
}
template <typename F>
QCH_HD double np_pairwise(const F& f, int n) {
  if (n <= 128) return np_pairwise_block(f, 0, n);
  return np_pairwise_rec(f, 0, n);
}

// ---------------------------------------------------------------------------
// NPAD selection key: reference ordering lexsort((r, c, -mag)) (npad.py:313-314)
// = larger magnitude first, then smaller column c (= i), then smaller row r (= j).
struct SelKey {
  double mag;  // < 0 means "no relevant entry"
  int c, r;
};
QCH_HD SelKey selkey_none() {
  SelKey k;
  k.mag = -1.0;
  k.c = 0x7fffffff;
  k.r = 0x7fffffff;
  return k;
}
QCH_HD bool selkey_better(const SelKey& a, const SelKey& b) {
  if (a.mag != b.mag) return a.mag > b.mag;
  if (a.c != b.c) return a.c < b.c;
  return a.r < b.r;
}

// Givens rotation parameters, npad.py:101-123 and _block_params npad.py:126-128.
struct RotParams {
  double cos_half, sin_half, phase;
  cplx s;  // block [[c, -conj(s)], [s, c]], s = -sin_half * exp(i*phase)
  int degenerate;
};

QCH_HD RotParams givens_params(cplx v, double hii_re, double hjj_re) {
  RotParams p;
  double g = hypot_cr(v.re, v.im);
  double phi = atan2(v.im, v.re);
  double delta = QDIV(QSUB(hii_re, hjj_re), 2.0);
  double r = hypot_cr(delta, g);
  double sgn = (delta >= 0.0) ? 1.0 : -1.0;
  double cos_t = QDIV(fabs(delta), r);
  double sin_t = QDIV(QMUL(sgn, g), r);
  double ch = QSQRT(QDIV(QADD(1.0, cos_t), 2.0));
  double sh = QDIV(sin_t, QMUL(2.0, ch));
  p.cos_half = ch;
  p.sin_half = sh;
  p.phase = phi;
  p.degenerate = (delta == 0.0);
  double sn, cs;
#ifdef __CUDA_ARCH__
  sincos(phi, &sn, &cs);
#else
  sn = sin(phi);
  cs = cos(phi);
#endif
  // -sin_half * exp(1j*phase): float promoted to complex, exact products
  p.s = np_rmul(-sh, mkc(cs, sn));
  return p;
}

// New 2x2 cross block of _conjugate_dense (npad.py:131-145): rows first, then
// columns on the updated rows, then the Hermitian pin.
struct Block2 {
  cplx ii, ij, ji, jj;
};
QCH_HD Block2 rotate_block(double c, cplx s, cplx hii, cplx hij, cplx hji, cplx hjj) {
  cplx sc = cconj(s);
  // row step
  cplx aii = csub(np_rmul(c, hii), np_cmul(sc, hji));
  cplx aij = csub(np_rmul(c, hij), np_cmul(sc, hjj));
  cplx aji = cadd(np_cmul(s, hii), np_rmul(c, hji));
  cplx ajj = cadd(np_cmul(s, hij), np_rmul(c, hjj));
  // column step
  Block2 o;
  o.ii = csub(np_rmul(c, aii), np_cmul(s, aij));
  o.ji = csub(np_rmul(c, aji), np_cmul(s, ajj));
  o.ij = cadd(np_cmul(sc, aii), np_rmul(c, aij));
  o.jj = cadd(np_cmul(sc, aji), np_rmul(c, ajj));
  // pin
  o.ii.im = 0.0;
  o.jj.im = 0.0;
  o.ji = cconj(o.ij);
  return o;
}

// row update of one column x: (new r_i[x], new r_j[x])
QCH_HD void rotate_rows(double c, cplx s, cplx ri, cplx rj, cplx* ni, cplx* nj) {
  *ni = csub(np_rmul(c, ri), np_cmul(cconj(s), rj));
  *nj = cadd(np_cmul(s, ri), np_rmul(c, rj));
}
// column update of one row x on (already row-updated, i.e. untouched) ci, cj
QCH_HD void rotate_cols(double c, cplx s, cplx ci, cplx cj, cplx* ni, cplx* nj) {
  *ni = csub(np_rmul(c, ci), np_cmul(s, cj));
  *nj = cadd(np_cmul(cconj(s), ci), np_rmul(c, cj));
}
