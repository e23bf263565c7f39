// magnus_small.cuh — per-interval Magnus arithmetic for small N (register
// matrices): coefficients (magnus.py:151-169 + SURVEY.md App. B), Taylor
// exp(-iH) (expm.py:56-71), propagator validation (expm.py:40-47).  Shared by
// the multi-kernel pipeline (magnus.cu) and the single-pass fused kernel
// (magnus_fused.cu).
#pragma once
#include "qch_internal.h"
#include "qch_math.cuh"

namespace qch {

constexpr int kTaylorOrder = 18;     // expm.py:19
constexpr double kScaleTarget = 0.5;  // expm.py:20

// ----------------------------------------------------------------------------
// Coefficients.  First order: magnus.py:164-168 (numpy pairwise sum of
// (left+right) then * dt/2).  Second order: SURVEY.md Appendix B.
struct CoefArgs {
  const double* sig;  // (K, S)
  int K;
  int64_t S;
  int64_t M;
  int sub;
  double dt;
};

__device__ __forceinline__ void interval_coeffs(const CoefArgs& a, int64_t n, int order, double* c1, double* c2) {
  const int K = a.K, sub = a.sub;
  const double h = a.dt;
  for (int k = 0; k < K; ++k) {
    const double* u = a.sig + (int64_t)k * a.S + n * sub;
    auto f = [&](int q) { return QADD(u[q], u[q + 1]); };
    c1[k] = QMUL(QDIV(h, 2.0), np_pairwise(f, sub));
  }
  if (order < 2) return;
  const double hh6 = QDIV(QMUL(h, h), 6.0);
  const double h2 = QDIV(h, 2.0);
  // alpha_k = sum_a [h*S_k(a) - a*h*tau_ak] - (h^2/6) sum_a (u_{a+1} - u_a)
  for (int k = 0; k < K; ++k) {
    const double* u = a.sig + (int64_t)k * a.S + n * sub;
    double run = 0.0, acc = 0.0, lin = 0.0;
    for (int q = 0; q < sub; ++q) {
      double tau = QMUL(h2, QADD(u[q], u[q + 1]));
      acc = QADD(acc, QSUB(QMUL(h, run), QMUL(QMUL((double)q, h), tau)));
      lin = QADD(lin, QSUB(u[q + 1], u[q]));
      run = QADD(run, tau);
    }
    c2[k] = QSUB(acc, QMUL(hh6, lin));
  }
  // beta_kl = sum_a [tau_ak S_l(a) - tau_al S_k(a)] - (h^2/6) sum_a (u_k,a u_l,a+1 - u_l,a u_k,a+1)
  int idx = K;
  for (int k = 0; k < K; ++k)
    for (int l = k + 1; l < K; ++l) {
      const double* uk = a.sig + (int64_t)k * a.S + n * sub;
      const double* ul = a.sig + (int64_t)l * a.S + n * sub;
      double sk = 0.0, sl = 0.0, acc = 0.0, cr = 0.0;
      for (int q = 0; q < sub; ++q) {
        double tk = QMUL(h2, QADD(uk[q], uk[q + 1]));
        double tl = QMUL(h2, QADD(ul[q], ul[q + 1]));
        acc = QADD(acc, QSUB(QMUL(tk, sl), QMUL(tl, sk)));
        cr = QADD(cr, QSUB(QMUL(uk[q], ul[q + 1]), QMUL(ul[q], uk[q + 1])));
        sk = QADD(sk, tk);
        sl = QADD(sl, tl);
      }
      c2[idx++] = QSUB(acc, QMUL(hh6, cr));
    }
}

// the same coefficients one at a time (no local arrays in the hot kernel)
__device__ __forceinline__ double coef1(const CoefArgs& a, int64_t n, int k) {
  const double* u = a.sig + (int64_t)k * a.S + n * a.sub;
  auto f = [&](int q) { return QADD(u[q], u[q + 1]); };
  return QMUL(QDIV(a.dt, 2.0), np_pairwise(f, a.sub));
}
__device__ __forceinline__ double coef_alpha(const CoefArgs& a, int64_t n, int k) {
  const double h = a.dt, h2 = QDIV(h, 2.0), hh6 = QDIV(QMUL(h, h), 6.0);
  const double* u = a.sig + (int64_t)k * a.S + n * a.sub;
  double run = 0.0, acc = 0.0, lin = 0.0;
  for (int q = 0; q < a.sub; ++q) {
    double tau = QMUL(h2, QADD(u[q], u[q + 1]));
    acc = QADD(acc, QSUB(QMUL(h, run), QMUL(QMUL((double)q, h), tau)));
    lin = QADD(lin, QSUB(u[q + 1], u[q]));
    run = QADD(run, tau);
  }
  return QSUB(acc, QMUL(hh6, lin));
}
__device__ __forceinline__ double coef_beta(const CoefArgs& a, int64_t n, int k, int l) {
  const double h = a.dt, h2 = QDIV(h, 2.0), hh6 = QDIV(QMUL(h, h), 6.0);
  const double* uk = a.sig + (int64_t)k * a.S + n * a.sub;
  const double* ul = a.sig + (int64_t)l * a.S + n * a.sub;
  double sk = 0.0, sl = 0.0, acc = 0.0, cr = 0.0;
  for (int q = 0; q < a.sub; ++q) {
    double tk = QMUL(h2, QADD(uk[q], uk[q + 1]));
    double tl = QMUL(h2, QADD(ul[q], ul[q + 1]));
    acc = QADD(acc, QSUB(QMUL(tk, sl), QMUL(tl, sk)));
    cr = QADD(cr, QSUB(QMUL(uk[q], ul[q + 1]), QMUL(ul[q], uk[q + 1])));
    sk = QADD(sk, tk);
    sl = QADD(sl, tl);
  }
  return QSUB(acc, QMUL(hh6, cr));
}

constexpr int kMaxK = 8;


// ----------------------------------------------------------------------------
// small dense matrices in registers
template <int N>
struct Mat {
  cplx v[N][N];
};
template <int N>
__device__ __forceinline__ Mat<N> mat_eye() {
  Mat<N> m;
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) m.v[r][c] = mkc(r == c ? 1.0 : 0.0, 0.0);
  return m;
}
template <int N>
__device__ __forceinline__ Mat<N> mat_mul(const Mat<N>& a, const Mat<N>& b) {
  Mat<N> o;
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) {
      cplx acc = np_cmul(a.v[r][0], b.v[0][c]);
#pragma unroll
      for (int k = 1; k < N; ++k) acc = cadd(acc, np_cmul(a.v[r][k], b.v[k][c]));
      o.v[r][c] = acc;
    }
  return o;
}
template <int N>
__device__ __forceinline__ cplx mat_det(const Mat<N>& m);
template <>
__device__ __forceinline__ cplx mat_det<1>(const Mat<1>& m) {
  return m.v[0][0];
}
template <>
__device__ __forceinline__ cplx mat_det<2>(const Mat<2>& m) {
  return csub(np_cmul(m.v[0][0], m.v[1][1]), np_cmul(m.v[0][1], m.v[1][0]));
}
template <>
__device__ __forceinline__ cplx mat_det<3>(const Mat<3>& m) {
  cplx a = np_cmul(m.v[0][0], csub(np_cmul(m.v[1][1], m.v[2][2]), np_cmul(m.v[1][2], m.v[2][1])));
  cplx b = np_cmul(m.v[0][1], csub(np_cmul(m.v[1][0], m.v[2][2]), np_cmul(m.v[1][2], m.v[2][0])));
  cplx c = np_cmul(m.v[0][2], csub(np_cmul(m.v[1][0], m.v[2][1]), np_cmul(m.v[1][1], m.v[2][0])));
  return cadd(csub(a, b), c);
}
template <>
__device__ __forceinline__ cplx mat_det<4>(const Mat<4>& m) {
  cplx acc = mkc(0, 0);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    Mat<3> s;
#pragma unroll
    for (int r = 1; r < 4; ++r) {
      int cc = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q != c) s.v[r - 1][cc++] = m.v[r][q];
    }
    cplx t = np_cmul(m.v[0][c], mat_det<3>(s));
    acc = (c & 1) ? csub(acc, t) : cadd(acc, t);
  }
  return acc;
}

// _expm_minus_i (expm.py:56-71) on one register matrix (hbar -> U)
template <int N>
__device__ __forceinline__ Mat<N> expm_minus_i_reg(const Mat<N>& hb) {
  Mat<N> a;
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) a.v[r][c] = mkc(hb.v[r][c].im, -hb.v[r][c].re);  // -1j * H, exact
  double norm = 0.0;
#pragma unroll
  for (int r = 0; r < N; ++r) {
    double rs = 0.0;  // numpy sequential sum for n < 8
#pragma unroll
    for (int c = 0; c < N; ++c) rs = QADD(rs, np_cabs(a.v[r][c]));
    norm = fmax(norm, rs);
  }
  int s = 0;
  if (norm > kScaleTarget) {
    s = (int)ceil(log2(QDIV(norm, kScaleTarget)));
    double scl = ldexp(1.0, -s);  // a / 2**s == a * 2**-s exactly
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c < N; ++c) a.v[r][c] = mkc(QMUL(a.v[r][c].re, scl), QMUL(a.v[r][c].im, scl));
  }
  Mat<N> out = mat_eye<N>(), term = mat_eye<N>();
  for (int k = 1; k <= kTaylorOrder; ++k) {
    term = mat_mul<N>(term, a);
    double inv = QDIV(1.0, (double)k);
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        term.v[r][c] = mkc(QMUL(term.v[r][c].re, inv), QMUL(term.v[r][c].im, inv));
        out.v[r][c] = cadd(out.v[r][c], term.v[r][c]);
      }
  }
  for (int q = 0; q < s; ++q) out = mat_mul<N>(out, out);
  return out;
}

// UnitaryPropagator.validate (expm.py:40-47)
template <int N>
__device__ __forceinline__ bool validate_reg(const Mat<N>& u) {
  double d2 = 0.0;
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) {
      cplx acc = mkc(0, 0);
#pragma unroll
      for (int k = 0; k < N; ++k) acc = cadd(acc, np_cmul(u.v[r][k], cconj(u.v[c][k])));
      double re = acc.re - (r == c ? 1.0 : 0.0);
      d2 += re * re + acc.im * acc.im;
    }
  double defect = sqrt(d2);
  if (!(defect <= 1e-10 * N)) return false;
  cplx d = mat_det<N>(u);
  double ad = hypot_cr(d.re, d.im);
  return fabs(ad - 1.0) <= 1e-8;
}

struct SmallArgs {
  CoefArgs ca;
  const double2* h0;    // (N,N)
  const double2* hk;    // (K,N,N)
  const double2* comm;  // (K + K(K-1)/2, N, N) (order 2)
  int order;
  double dt_int;
  int check;
  double2* ubuf;    // (M,N,N) propagators (the caller's props buffer when requested)
  double2* runp;    // (nruns,N,N) block-exclusive prefix of each run
  double2* agg;     // (nblocks, N, N) block aggregates -> exclusive block prefixes
  unsigned long long* bad;  // [0] first non-unitary interval, [1] first norm drift
};

template <int N>
__device__ __forceinline__ void ld_mat(Mat<N>& m, const double2* p) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) m.v[r][c] = d2c(p[r * N + c]);
}
template <int N>
__device__ __forceinline__ void st_mat(double2* p, const Mat<N>& m) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) p[r * N + c] = c2d(m.v[r][c]);
}

// complex matrix product with FMA accumulation (the BLAS-like rounding of the
// reference's `term @ a`, expm.py:67; 4 FMA per complex MAC)
template <int N>
__device__ __forceinline__ Mat<N> mat_mul_fma(const Mat<N>& a, const Mat<N>& b) {
  Mat<N> o;
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) {
      double re = a.v[r][0].re * b.v[0][c].re;
      double im = a.v[r][0].re * b.v[0][c].im;
      re = fma(-a.v[r][0].im, b.v[0][c].im, re);
      im = fma(a.v[r][0].im, b.v[0][c].re, im);
#pragma unroll
      for (int k = 1; k < N; ++k) {
        re = fma(a.v[r][k].re, b.v[k][c].re, re);
        im = fma(a.v[r][k].re, b.v[k][c].im, im);
        re = fma(-a.v[r][k].im, b.v[k][c].im, re);
        im = fma(a.v[r][k].im, b.v[k][c].re, im);
      }
      o.v[r][c] = mkc(re, im);
    }
  return o;
}

// Truncation degree table for the Taylor series of exp(a), ||a|| <= nu:
// kTheta[m] is the largest nu with 2 nu^(m+1)/(m+1)! <= 2^-56, so the series
// cut after degree m differs from the full series (and from the reference's
// 18-term sum, expm.py:66-68) by < 1.4e-17 relative to ||exp(a)|| = 1.
static __constant__ double kTheta[19] = {
    6.9388939039072284e-18, 3.7252902984619141e-09, 3.4658824783938236e-06, 0.00011359922596461176,
    0.00096403832316153276, 0.0041346344980966003,  0.011958436387519561,   0.026968161873314821,
    0.051431375833317965,   0.087117484748903212,   0.13524818677402944,    0.19654813817446753,
    0.27133475643086408,    0.3596131914026986,     0.46116109021995333,    0.57559811770713287,
    0.70244016939905507,    0.84114022780138098,    0.99111835560814376};
static __constant__ double kInvFact[20] = {1.0,
                                    1.0,
                                    0.5,
                                    0.16666666666666666,
                                    0.041666666666666664,
                                    0.008333333333333333,
                                    0.001388888888888889,
                                    0.0001984126984126984,
                                    2.48015873015873e-05,
                                    2.7557319223985893e-06,
                                    2.755731922398589e-07,
                                    2.505210838544172e-08,
                                    2.08767569878681e-09,
                                    1.6059043836821613e-10,
                                    1.1470745597729725e-11,
                                    7.647163731819816e-13,
                                    4.779477332387385e-14,
                                    2.8114572543455206e-15,
                                    1.5619206968586225e-16,
                                    0.0};

// _expm_minus_i (expm.py:56-71) in registers.  Same scaling as the reference
// (s from numpy's max row sum of |a|, target 0.5), evaluated faster:
//  * the scaling test uses the cheap bound sum(|re|+|im|) >= the reference's
//    norm (up to rounding, 1e-12 margin); only when it could exceed 0.5 is the
//    exact numpy norm computed, so s is always the reference's s;
//  * the Taylor polynomial is cut at the degree m whose remainder is provably
//    < 2^-56 (kTheta; m = 6-7 for the config-2 intervals, <= 15 after
//    scaling) and evaluated by Paterson-Stockmeyer/Horner in a^2:
//      p(a) = sum_j (a^2)^j (c_2j I + c_2j+1 a),   c_k = 1/k!
//    i.e. 1 + m/2 matrix products instead of the reference's 17.
// The result agrees with the reference's to rounding (~1e-16), inside the
// 1e-10 parity bar.
template <int N>
__device__ __forceinline__ Mat<N> expm_minus_i_fast(const Mat<N>& hb) {
  Mat<N> a;
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) a.v[r][c] = mkc(hb.v[r][c].im, -hb.v[r][c].re);
  double nb = 0.0;  // upper bound of the infinity norm
#pragma unroll
  for (int r = 0; r < N; ++r) {
    double rs = 0.0;
#pragma unroll
    for (int c = 0; c < N; ++c) rs += fabs(a.v[r][c].re) + fabs(a.v[r][c].im);
    nb = fmax(nb, rs);
  }
  int s = 0;
  if (!(nb * (1.0 + 1e-12) <= kScaleTarget)) {  // (also catches NaN)
    double norm = 0.0;
#pragma unroll
    for (int r = 0; r < N; ++r) {
      double rs = 0.0;
#pragma unroll
      for (int c = 0; c < N; ++c) rs = QADD(rs, np_cabs(a.v[r][c]));
      norm = fmax(norm, rs);
    }
    if (norm > kScaleTarget) {
      s = (int)ceil(log2(QDIV(norm, kScaleTarget)));
      const double scl = ldexp(1.0, -s);
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int c = 0; c < N; ++c) a.v[r][c] = mkc(a.v[r][c].re * scl, a.v[r][c].im * scl);
      nb *= scl;
    }
  }
  // smallest degree m >= 1 with nb > kTheta[m-1] (kTheta increasing): count
  // the thresholds below nb with independent compares (a dependent
  // compare-and-load loop sat on the critical path of every interval)
  int m = 0;
#pragma unroll
  for (int q = 0; q < kTaylorOrder; ++q) m += nb > kTheta[q] ? 1 : 0;
  m = max(m, 1);
  if (!(nb == nb)) m = kTaylorOrder;
  const Mat<N> a2 = mat_mul_fma<N>(a, a);
  int j = m >> 1;
  Mat<N> acc;
  {
    const double c0 = kInvFact[2 * j], c1 = kInvFact[2 * j + 1] * (2 * j + 1 <= m ? 1.0 : 0.0);
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c < N; ++c)
        acc.v[r][c] = mkc(fma(c1, a.v[r][c].re, r == c ? c0 : 0.0), c1 * a.v[r][c].im);
  }
#pragma unroll 1
  for (--j; j >= 0; --j) {
    const double c0 = kInvFact[2 * j], c1 = kInvFact[2 * j + 1];
    // column c of a2*acc depends on column c of acc only: update in place
#pragma unroll
    for (int c = 0; c < N; ++c) {
      cplx col[N];
#pragma unroll
      for (int r = 0; r < N; ++r) {
        double re = fma(c1, a.v[r][c].re, r == c ? c0 : 0.0);
        double im = c1 * a.v[r][c].im;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          re = fma(a2.v[r][k].re, acc.v[k][c].re, re);
          re = fma(-a2.v[r][k].im, acc.v[k][c].im, re);
          im = fma(a2.v[r][k].re, acc.v[k][c].im, im);
          im = fma(a2.v[r][k].im, acc.v[k][c].re, im);
        }
        col[r] = mkc(re, im);
      }
#pragma unroll
      for (int r = 0; r < N; ++r) acc.v[r][c] = col[r];
    }
  }
#pragma unroll 1
  for (int q = 0; q < s; ++q) acc = mat_mul_fma<N>(acc, acc);
  return acc;
}



// Shared-memory operator table of a block: H0 | H_k (K) | basis commutators
// (order 2: [H0,H_k] then [H_k,H_l], k<l).  When g.comm is null the
// commutators are formed here as [A,B] = AB - (AB)^dag (A, B Hermitian).
template <int N>
__device__ __forceinline__ void load_ops(const SmallArgs& g, double2* s_ops, const double2* h0 = nullptr,
                                         const double2* hk = nullptr) {
  const int K = g.ca.K;
  const int ncomm = K + K * (K - 1) / 2;
  if (h0 == nullptr) h0 = g.h0;
  if (hk == nullptr) hk = g.hk;
  for (int q = threadIdx.x; q < N * N; q += blockDim.x) s_ops[q] = h0[q];
  for (int q = threadIdx.x; q < K * N * N; q += blockDim.x) s_ops[N * N + q] = hk[q];
  if (g.order >= 2 && g.comm != nullptr)
    for (int q = threadIdx.x; q < ncomm * N * N; q += blockDim.x) s_ops[(1 + K) * N * N + q] = g.comm[q];
  __syncthreads();
  if (g.order >= 2 && g.comm == nullptr) {
    for (int q = threadIdx.x; q < ncomm * N * N; q += blockDim.x) {
      const int idx = q / (N * N), e = q % (N * N), r = e / N, c = e % N;
      int ka = 0, kb = 1 + idx;  // [H0, H_idx]
      if (idx >= K) {
        int t = idx - K;
        ka = 0;
        while (t >= K - 1 - ka) {
          t -= K - 1 - ka;
          ++ka;
        }
        kb = 1 + ka + 1 + t;
        ka = 1 + ka;
      }
      const double2* A = s_ops + ka * N * N;
      const double2* B = s_ops + kb * N * N;
      cplx p = mkc(0, 0), pt = mkc(0, 0);  // (AB)[r][c], (AB)[c][r]
#pragma unroll
      for (int k = 0; k < N; ++k) {
        p = cadd(p, np_cmul(d2c(A[r * N + k]), d2c(B[k * N + c])));
        pt = cadd(pt, np_cmul(d2c(A[c * N + k]), d2c(B[k * N + r])));
      }
      s_ops[(1 + K + idx) * N * N + e] = c2d(csub(p, cconj(pt)));
    }
    __syncthreads();
  }
}

// real scalar times complex.  numpy promotes w to (w + 0j) and multiplies
// with FMAs; for finite operands that is exactly (w*re, w*im) rounded once
// each, which is what this computes in 2 instead of 4 instructions.
__device__ __forceinline__ cplx rmul(double w, cplx b) { return mkc(QMUL(w, b.re), QMUL(w, b.im)); }

// Hbar_n for interval n (magnus.py:185-189: h = dt*drift; h = h + w*ctrl,
// numpy order) plus, for order 2, (-i/2) X_n with X_n = sum alpha [H0,H_k] +
// sum beta [H_k,H_l].
template <int N>
__device__ __forceinline__ Mat<N> interval_hbar(const SmallArgs& g, const double2* s_ops, int64_t n) {
  const int K = g.ca.K;
  Mat<N> hb;
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) hb.v[r][c] = rmul(g.dt_int, d2c(s_ops[r * N + c]));
  for (int k = 0; k < K; ++k) {
    const double w = coef1(g.ca, n, k);
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c < N; ++c) hb.v[r][c] = cadd(hb.v[r][c], rmul(w, d2c(s_ops[(1 + k) * N * N + r * N + c])));
  }
  if (g.order >= 2) {
    Mat<N> x;
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c < N; ++c) x.v[r][c] = mkc(0, 0);
    int q = 0;
    for (int k = 0; k < K; ++k, ++q) {
      const double w = coef_alpha(g.ca, n, k);
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int c = 0; c < N; ++c)
          x.v[r][c] = cadd(x.v[r][c], rmul(w, d2c(s_ops[(1 + K + q) * N * N + r * N + c])));
    }
    for (int k = 0; k < K; ++k)
      for (int l = k + 1; l < K; ++l, ++q) {
        const double w = coef_beta(g.ca, n, k, l);
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int c = 0; c < N; ++c)
            x.v[r][c] = cadd(x.v[r][c], rmul(w, d2c(s_ops[(1 + K + q) * N * N + r * N + c])));
      }
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c < N; ++c) hb.v[r][c] = cadd(hb.v[r][c], mkc(QMUL(0.5, x.v[r][c].im), QMUL(-0.5, x.v[r][c].re)));
  }
  return hb;
}

// interval_hbar for a compile-time samples-per-interval SUB with the signal
// window in shared memory (the fused kernel's staged window; `sig` must point
// into shared memory so the loads are LDS): each control's SUB+1 samples are
// loaded once into registers and the coefficients are formed from them with
// exactly the operation order of coef1 / coef_alpha / coef_beta.
template <int N, int SUB>
__device__ __forceinline__ Mat<N> interval_hbar_fixed(const SmallArgs& g, const double2* s_ops, const double* sig,
                                                      int64_t S, int64_t nl) {
  const int K = g.ca.K;
  const double h = g.ca.dt, h2 = QDIV(h, 2.0), hh6 = QDIV(QMUL(h, h), 6.0);
  Mat<N> hb, x;
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) {
      hb.v[r][c] = rmul(g.dt_int, d2c(s_ops[r * N + c]));
      x.v[r][c] = mkc(0, 0);
    }
  const bool o2 = g.order >= 2;
  for (int k = 0; k < K; ++k) {
    double u[SUB + 1];
#pragma unroll
    for (int q = 0; q <= SUB; ++q) u[q] = sig[k * S + nl * SUB + q];
    const double w = QMUL(h2, np_pairwise([&](int q) { return QADD(u[q], u[q + 1]); }, SUB));
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c < N; ++c) hb.v[r][c] = cadd(hb.v[r][c], rmul(w, d2c(s_ops[(1 + k) * N * N + r * N + c])));
    if (o2) {
      double run = 0.0, acc = 0.0, lin = 0.0;
#pragma unroll
      for (int q = 0; q < SUB; ++q) {
        const double tau = QMUL(h2, QADD(u[q], u[q + 1]));
        acc = QADD(acc, QSUB(QMUL(h, run), QMUL(QMUL((double)q, h), tau)));
        lin = QADD(lin, QSUB(u[q + 1], u[q]));
        run = QADD(run, tau);
      }
      const double a = QSUB(acc, QMUL(hh6, lin));
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int c = 0; c < N; ++c)
          x.v[r][c] = cadd(x.v[r][c], rmul(a, d2c(s_ops[(1 + K + k) * N * N + r * N + c])));
    }
  }
  if (o2) {
    int q2 = K;
    for (int k = 0; k < K; ++k) {
      double uk[SUB + 1];
#pragma unroll
      for (int q = 0; q <= SUB; ++q) uk[q] = sig[k * S + nl * SUB + q];
      for (int l = k + 1; l < K; ++l, ++q2) {
        double ul[SUB + 1];
#pragma unroll
        for (int q = 0; q <= SUB; ++q) ul[q] = sig[l * S + nl * SUB + q];
        double sk = 0.0, sl = 0.0, acc = 0.0, cr = 0.0;
#pragma unroll
        for (int q = 0; q < SUB; ++q) {
          const double tk = QMUL(h2, QADD(uk[q], uk[q + 1]));
          const double tl = QMUL(h2, QADD(ul[q], ul[q + 1]));
          acc = QADD(acc, QSUB(QMUL(tk, sl), QMUL(tl, sk)));
          cr = QADD(cr, QSUB(QMUL(uk[q], ul[q + 1]), QMUL(ul[q], uk[q + 1])));
          sk = QADD(sk, tk);
          sl = QADD(sl, tl);
        }
        const double b = QSUB(acc, QMUL(hh6, cr));
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int c = 0; c < N; ++c)
            x.v[r][c] = cadd(x.v[r][c], rmul(b, d2c(s_ops[(1 + K + q2) * N * N + r * N + c])));
      }
    }
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c < N; ++c) hb.v[r][c] = cadd(hb.v[r][c], mkc(QMUL(0.5, x.v[r][c].im), QMUL(-0.5, x.v[r][c].re)));
  }
  return hb;
}

template <int N>
__host__ __device__ constexpr size_t ops_smem_bytes(int K, int order) {
  return sizeof(double2) * (size_t)(1 + K + (order >= 2 ? K + K * (K - 1) / 2 : 0)) * N * N;
}

}  // namespace qch
