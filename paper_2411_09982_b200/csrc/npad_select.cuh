// npad_select.cuh — exact coupling selection with cheap keys.
//
// The reference picks the pivot by numpy's |z| = L*sqrt(fma(S/L,S/L,1))
// (operators.py:133-139, npad.py:313-317), ties broken by (i, j).  Computing
// that for every candidate costs a correctly-rounded divide and square root
// (~40 FP64 instructions, ~250 cycles of latency).  Instead each candidate
// carries key q = re^2 + im^2 (2 instructions).  q is within 2 ulp of |z|^2 and
// numpy's |z| within 2 ulp of |z|, so whenever two keys differ by more than a
// relative kRel = 1e-12 the q-order IS the |z|-order; inside that band the
// exact numpy magnitude m is computed (lazily, cached in the candidate) and
// compared with the reference tie-break.  The result is the reference's pick,
// bit for bit, at a fraction of the cost.  (Matrices whose relevant entries
// could underflow/overflow q run with exact keys: q := m.)
//
// Warp argmax uses redux.sync on the two halves of q's bit pattern (monotone
// for non-negative doubles) plus one ballot: ~6 instructions when the winner
// is clear, a shuffle reduction over the near-tie lanes otherwise.
#pragma once
#include "qch_math.cuh"

namespace qch {

constexpr double kRel = 1e-12;
constexpr unsigned kFull = 0xffffffffu;

struct Cand {
  double q;     // key (> 0); <= 0 means none
  double m;     // exact numpy |z| or -1 if not computed yet
  unsigned cr;  // (c << 16) | r of the lower-triangle entry (tie-break order)
  double2 v;    // the lower-triangle entry H[r, c]
};

__device__ __forceinline__ Cand cand_none() {
  Cand c;
  c.q = 0.0;
  c.m = -1.0;
  c.cr = 0xffffffffu;
  c.v = make_double2(0.0, 0.0);
  return c;
}

// out-of-line exact magnitude: the rare path must not bloat the hot loops
// (the instruction cache is the first limiter of these kernels)
static __device__ __noinline__ double np_cabs_ool(double re, double im) { return np_cabs(re, im); }

__device__ __forceinline__ double key_of(double2 v, bool ek) {
  return ek ? np_cabs_ool(v.x, v.y) : fma(v.x, v.x, v.y * v.y);
}

__device__ __forceinline__ Cand make_cand(double2 v, unsigned cr, bool ek) {
  Cand c;
  c.q = key_of(v, ek);
  c.m = ek ? c.q : -1.0;
  c.cr = cr;
  c.v = v;
  return c;
}

__device__ __forceinline__ double cand_m(Cand& a) {
  if (a.m < 0.0) a.m = np_cabs_ool(a.v.x, a.v.y);
  return a.m;
}

// near-tie resolution with exact numpy magnitudes (out of line; operands by
// value so the callers' candidates stay in registers)
static __device__ __noinline__ bool cand_better_exact_v(double2 av, double am, unsigned acr, double2 bv, double bm,
                                                        unsigned bcr) {
  if (am < 0.0) am = np_cabs(av.x, av.y);
  if (bm < 0.0) bm = np_cabs(bv.x, bv.y);
  if (am != bm) return am > bm;
  return acr < bcr;
}

// a strictly before b in the reference order (mag desc, c asc, r asc)
// (none = q 0: 'a.q > b.q (1 + kRel)' already orders none below any
// candidate and two nones as equal; one branch, taken only inside the band)
__device__ __forceinline__ bool cand_better(const Cand& a, const Cand& b) {
  const bool gt = a.q > b.q * (1.0 + kRel);
  const bool lt = b.q > a.q * (1.0 + kRel);
  if (gt || lt || !(a.q > 0.0) || !(b.q > 0.0)) return gt;
  return cand_better_exact_v(a.v, a.m, a.cr, b.v, b.m, b.cr);
}

__device__ __forceinline__ void cand_take(Cand& best, const Cand& c) {
  if (cand_better(c, best)) best = c;
}

static __device__ __noinline__ int warp_argmax_exact(double2 v, double m0, unsigned cr0, bool nearf) {
  double m = -1.0;
  unsigned cr = 0xffffffffu;
  double mine = -1.0;
  if (nearf) {
    mine = (m0 < 0.0) ? np_cabs(v.x, v.y) : m0;
    m = mine;
    cr = cr0;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    double om = __shfl_xor_sync(kFull, m, off);
    unsigned ocr = __shfl_xor_sync(kFull, cr, off);
    if (om > m || (om == m && ocr < cr)) {
      m = om;
      cr = ocr;
    }
  }
  const unsigned w = __ballot_sync(kFull, nearf && mine == m && cr0 == cr);
  return __ffs(w) - 1;
}

// winner lane of the warp (all lanes agree), -1 if no lane has a candidate.
__device__ __forceinline__ int warp_argmax(Cand& c) {
  const unsigned long long b = (c.q > 0.0) ? (unsigned long long)__double_as_longlong(c.q) : 0ull;
  const unsigned hi = (unsigned)(b >> 32);
  const unsigned hmax = __reduce_max_sync(kFull, hi);
  if (hmax == 0u) return -1;
  const unsigned lo = (hi == hmax) ? (unsigned)b : 0u;
  const unsigned lmax = __reduce_max_sync(kFull, lo);
  const double qs = __longlong_as_double((long long)(((unsigned long long)hmax << 32) | lmax));
  const bool nearf = (c.q > 0.0) && (c.q >= qs * (1.0 - kRel));
  const unsigned near = __ballot_sync(kFull, nearf);
  if (__popc(near) == 1) return __ffs(near) - 1;
  return warp_argmax_exact(c.v, c.m, c.cr, nearf);
}

// Rotation scalars for the device loop: same mathematics as
// givens_rotation_matrix + _block_params (npad.py:101-128) with two
// transcendental steps instead of hypot/atan2/sincos:
//   r = sqrt(delta^2 + g^2),  w = 2 r (r + |delta|),
//   cos(t/2) = (r + |delta|)/sqrt(w),  s = -sign(delta) v / sqrt(w)
// (s = -sin(t/2) e^{i phi} with e^{i phi} = v/g).  Agrees with the
// reference's scalars to a few ulp; the pivot sequence is unaffected (the
// parity tests check it bit for bit).
__device__ __forceinline__ void givens_fast(cplx v, double hii, double hjj, double* c, cplx* s) {
  const double delta = QMUL(QSUB(hii, hjj), 0.5);
  const double g2 = fma(v.re, v.re, v.im * v.im);
  const double r = sqrt(fma(delta, delta, g2));
  const double ad = fabs(delta);
  const double rpa = r + ad;
  const double rs = rsqrt(2.0 * r * rpa);
  const double sg = (delta >= 0.0) ? -rs : rs;
  *c = rpa * rs;
  *s = mkc(sg * v.re, sg * v.im);
}

}  // namespace qch
