// npad_fullwarp.cu — full-diagonal npad_run (npad.py:320-354) for small
// dimensions (n <= 64, BASELINE config 1: dim 60) with ONE WARP per chain.
//
// The single-CTA rows kernel (npad_run.cu) spends three block barriers and a
// shared-memory candidate exchange per rotation; at n = 60 its 2 warps are
// idle most of the time.  Here one warp owns the whole chain:
//  * the matrix lives in shared memory (row pitch 65 elements, so a 16-byte
//    column walk touches 8 distinct bank groups);
//  * lane l owns rows l and l + 32: their best candidate (strict lower
//    triangle, the reference's order: certified |z|^2 key, exact numpy |z|
//    near ties, then (c, r)) stays in registers;
//  * a rotation (i, j): warp argmax of the row bests (shuffles), the Givens
//    scalars and the 2x2 block computed redundantly by every lane (no
//    broadcast), rows i, j rotated with lane l handling columns l, l + 32 and
//    the mirrored columns written as conjugates (bitwise-Hermitian input), the
//    new rows i, j reduced from registers, every other row folding its two new
//    entries — and rows whose argmax column was i or j rescanned by the whole
//    warp (one warp argmax per row).
// Same arithmetic as _conjugate_dense (qch_math.cuh), same pivots as the
// reference; the state (row bests) is persisted in the rows kernel's format,
// so the two drivers are interchangeable mid-chain.
#include <cstdlib>
#include <cstring>

#include "npad_run.h"
#include "npad_select.cuh"
#include "qch_internal.h"

namespace qch {
namespace {

constexpr int kPitch = 65;  // shared-memory row pitch (complex elements)
constexpr int kMaxN = 64;

__device__ __forceinline__ bool below_thr_fw(const Cand& p, double thr, bool ek) {
  // mag < threshold with mag the exact numpy |z| (npad.py:348)
  if (ek) return p.q < thr;
  const double t2 = thr * thr;
  if (p.q > t2 * (1.0 + kRel)) return false;
  if (p.q < t2 * (1.0 - kRel)) return true;
  return np_cabs_ool(p.v.x, p.v.y) < thr;
}

__device__ __forceinline__ Cand shfl_cand(const Cand& c, int src) {
  Cand o;
  o.q = __shfl_sync(kFull, c.q, src);
  o.m = __shfl_sync(kFull, c.m, src);
  o.cr = __shfl_sync(kFull, c.cr, src);
  o.v.x = __shfl_sync(kFull, c.v.x, src);
  o.v.y = __shfl_sync(kFull, c.v.y, src);
  return o;
}

// the warp's best candidate, in every lane (q <= 0: none).  (A butterfly of
// whole candidates through cand_better measured 1.7x slower per rotation
// than this REDUX-based argmax plus one broadcast.)
__device__ __forceinline__ Cand warp_best(Cand c) {
  const int wl = warp_argmax(c);
  if (wl < 0) return cand_none();
  return shfl_cand(c, wl);
}

// two independent warp argmaxes with their REDUX / ballot steps interleaved
// (same winners as two warp_best calls); the rare near-tie path stays exact
__device__ __forceinline__ void warp_best2(Cand& c1, Cand& c2) {
  const unsigned long long b1 = (c1.q > 0.0) ? (unsigned long long)__double_as_longlong(c1.q) : 0ull;
  const unsigned long long b2 = (c2.q > 0.0) ? (unsigned long long)__double_as_longlong(c2.q) : 0ull;
  const unsigned h1 = (unsigned)(b1 >> 32), h2 = (unsigned)(b2 >> 32);
  const unsigned hm1 = __reduce_max_sync(kFull, h1), hm2 = __reduce_max_sync(kFull, h2);
  const unsigned lm1 = __reduce_max_sync(kFull, (h1 == hm1) ? (unsigned)b1 : 0u);
  const unsigned lm2 = __reduce_max_sync(kFull, (h2 == hm2) ? (unsigned)b2 : 0u);
  const double qs1 = __longlong_as_double((long long)(((unsigned long long)hm1 << 32) | lm1));
  const double qs2 = __longlong_as_double((long long)(((unsigned long long)hm2 << 32) | lm2));
  const bool nf1 = (c1.q > 0.0) && (c1.q >= qs1 * (1.0 - kRel));
  const bool nf2 = (c2.q > 0.0) && (c2.q >= qs2 * (1.0 - kRel));
  const unsigned n1 = __ballot_sync(kFull, nf1), n2 = __ballot_sync(kFull, nf2);
  int w1 = -1, w2 = -1;
  if (hm1 != 0u) w1 = (__popc(n1) == 1) ? __ffs(n1) - 1 : warp_argmax_exact(c1.v, c1.m, c1.cr, nf1);
  if (hm2 != 0u) w2 = (__popc(n2) == 1) ? __ffs(n2) - 1 : warp_argmax_exact(c2.v, c2.m, c2.cr, nf2);
  const Cand o1 = shfl_cand(c1, w1 >= 0 ? w1 : 0), o2 = shfl_cand(c2, w2 >= 0 ? w2 : 0);
  c1 = w1 >= 0 ? o1 : cand_none();
  c2 = w2 >= 0 ? o2 : cand_none();
}

// EK: exact-magnitude keys (compile-time, so make_cand carries no branch)
template <bool EK, bool ST>  // ST: per-phase cycle counters (QCH_NPAD_STATS), compiled out otherwise
__global__ void __launch_bounds__(32) npad_full_warp_kernel(NpadJob2* __restrict__ jobs, NpadCommon2 cm) {
  extern __shared__ __align__(16) double2 hs[];  // n rows x kPitch
  NpadJob2* job = jobs + blockIdx.x;
  const int n = cm.n, lane = threadIdx.x;
  constexpr bool ek = EK;
  double2* hg = job->h;
  double2* ug = job->u;
  for (int r = 0; r < n; ++r)
    for (int x = lane; x < n; x += 32) hs[r * kPitch + x] = hg[(size_t)r * n + x];
  Cand rb[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int x = lane + 32 * q;
    rb[q] = cand_none();
    if (x < n && job->st_q[x] > 0.0) {
      rb[q].q = job->st_q[x];
      rb[q].cr = ((unsigned)job->st_c[x] << 16) | (unsigned)x;
      rb[q].v = job->st_v[x];
    }
  }
  __syncwarp();

  long long applied = job->applied;
  const double thr = job->threshold;
  int* const piv_log = job->pivots;  // loaded once (the stores through it could alias the job record)
  const long long piv_cap = job->pivot_cap;
  int status = 0;
  long long cyc[5] = {0, 0, 0, 0, 0}, nresc = 0;  // select, scalars, rotate, rows i/j, rescans
  long long c0 = clock64();
  while (true) {
    Cand best = rb[0];
    cand_take(best, rb[1]);
    const Cand piv = warp_best(best);
    if (applied >= cm.stop_at) {
      status = 2;
      break;
    }
    if (!(piv.q > 0.0) || below_thr_fw(piv, thr, ek)) {
      status = 0;
      break;
    }
    if (applied >= cm.max_iter) {
      status = 1;
      break;
    }
    long long c1 = 0;
    if (ST) {
      c1 = clock64();
      cyc[0] += c1 - c0;
    }
    const int i = (int)(piv.cr >> 16), j = (int)(piv.cr & 0xffffu);  // i < j
    const cplx v = d2c(piv.v);
    // rows i, j of this lane's columns, loaded before the scalars' long
    // sqrt / rsqrt chain so the loads overlap it
    double2 ri2[2], rj2[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int x = lane + 32 * q;
      ri2[q] = x < n ? hs[i * kPitch + x] : make_double2(0.0, 0.0);
      rj2[q] = x < n ? hs[j * kPitch + x] : make_double2(0.0, 0.0);
    }
    const double hii = hs[i * kPitch + i].x, hjj = hs[j * kPitch + j].x;
    double c;
    cplx s;
    givens_fast(v, hii, hjj, &c, &s);
    const Block2 blk = rotate_block(c, s, mkc(hii, 0.0), cconj(v), v, mkc(hjj, 0.0));
    if (lane == 0 && piv_log != nullptr && applied < piv_cap) {
      piv_log[2 * applied] = i;
      piv_log[2 * applied + 1] = j;
    }
    long long c2 = 0;
    if (ST) {
      c2 = clock64();
      cyc[1] += c2 - c1;
    }
    Cand pi = cand_none(), pj = cand_none();
    bool resc[2] = {false, false};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int x = lane + 32 * q;
      if (x >= n || x == i || x == j) continue;
      cplx ni, nj;
      rotate_rows(c, s, d2c(ri2[q]), d2c(rj2[q]), &ni, &nj);
      const cplx cxi = cconj(ni), cxj = cconj(nj);
      hs[i * kPitch + x] = c2d(ni);
      hs[j * kPitch + x] = c2d(nj);
      hs[x * kPitch + i] = c2d(cxi);
      hs[x * kPitch + j] = c2d(cxj);
      if (x < i) cand_take(pi, make_cand(c2d(ni), ((unsigned)x << 16) | (unsigned)i, ek));
      if (x < j) cand_take(pj, make_cand(c2d(nj), ((unsigned)x << 16) | (unsigned)j, ek));
      // row x: its entries at columns i and j changed
      const int col = rb[q].q > 0.0 ? (int)(rb[q].cr >> 16) : -1;
      if (col == i || col == j) {
        resc[q] = true;
      } else {
        if (i < x) cand_take(rb[q], make_cand(c2d(cxi), ((unsigned)i << 16) | (unsigned)x, ek));
        if (j < x) cand_take(rb[q], make_cand(c2d(cxj), ((unsigned)j << 16) | (unsigned)x, ek));
      }
    }
    if (ug != nullptr) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int x = lane + 32 * q;
        if (x >= n) continue;
        cplx ni, nj;
        rotate_rows(c, s, d2c(ug[(size_t)i * n + x]), d2c(ug[(size_t)j * n + x]), &ni, &nj);
        ug[(size_t)i * n + x] = c2d(ni);
        ug[(size_t)j * n + x] = c2d(nj);
      }
    }
    if (lane == 0) {
      hs[i * kPitch + i] = c2d(blk.ii);
      hs[i * kPitch + j] = c2d(blk.ij);
      hs[j * kPitch + i] = c2d(blk.ji);
      hs[j * kPitch + j] = c2d(blk.jj);
      cand_take(pj, make_cand(c2d(blk.ji), ((unsigned)i << 16) | (unsigned)j, ek));
    }
    long long c3 = 0;
    if (ST) {
      c3 = clock64();
      cyc[2] += c3 - c2;
    }
    // rows i, j: reduced from the fresh values
    Cand bi = pi, bj = pj;
    warp_best2(bi, bj);
    if (lane == (i & 31)) {
      if (i >> 5) rb[1] = bi;
      else rb[0] = bi;
    }
    if (lane == (j & 31)) {
      if (j >> 5) rb[1] = bj;
      else rb[0] = bj;
    }
    __syncwarp();  // the rotated rows / columns visible to the rescans
    // rows whose argmax column was i or j: whole-warp rescans
    unsigned m0 = __ballot_sync(kFull, resc[0]), m1 = __ballot_sync(kFull, resc[1]);
    long long c4 = 0;
    if (ST) {
      c4 = clock64();
      cyc[3] += c4 - c3;
      nresc += __popc(m0) + __popc(m1);
    }
    // two rows per pass (independent argmaxes, interleaved)
    auto next_row = [&]() {
      int r = -1;
      if (m0) {
        r = __ffs(m0) - 1;
        m0 &= m0 - 1;
      } else if (m1) {
        r = __ffs(m1) - 1 + 32;
        m1 &= m1 - 1;
      }
      return r;
    };
    while (m0 | m1) {
      const int r = next_row(), r2 = next_row();  // r2 = -1: one row left
      Cand b = cand_none(), b2 = cand_none();
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int x = lane + 32 * q;
        if (x < r) cand_take(b, make_cand(hs[r * kPitch + x], ((unsigned)x << 16) | (unsigned)r, ek));
        if (x < r2) cand_take(b2, make_cand(hs[r2 * kPitch + x], ((unsigned)x << 16) | (unsigned)r2, ek));
      }
      warp_best2(b, b2);
      if (lane == (r & 31)) {
        if (r >> 5) rb[1] = b;
        else rb[0] = b;
      }
      if (r2 >= 0 && lane == (r2 & 31)) {
        if (r2 >> 5) rb[1] = b2;
        else rb[0] = b2;
      }
    }
    ++applied;
    if (ST) {
      c0 = clock64();
      cyc[4] += c0 - c4;
    }
  }
  if (ST && lane == 0) {
    const double a = applied > 0 ? (double)applied : 1.0;
    printf("npad full-warp n=%d: %lld rotations, cycles/rotation select %.0f scalars %.0f rotate %.0f rows-ij %.0f "
           "rescans %.0f (%.2f rows)\n",
           n, applied, cyc[0] / a, cyc[1] / a, cyc[2] / a, cyc[3] / a, cyc[4] / a, nresc / a);
  }

  __syncwarp();
  for (int r = 0; r < n; ++r)
    for (int x = lane; x < n; x += 32) hg[(size_t)r * n + x] = hs[r * kPitch + x];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int x = lane + 32 * q;
    if (x < n) {
      job->st_q[x] = rb[q].q > 0.0 ? rb[q].q : 0.0;
      job->st_c[x] = rb[q].q > 0.0 ? (int)(rb[q].cr >> 16) : -1;
      job->st_v[x] = rb[q].v;
    }
  }
  if (lane == 0) {
    job->applied = applied;
    job->status = status;
  }
}

}  // namespace

// full-diagonal, bitwise-Hermitian chains of dimension <= 64: one warp each
bool npad_full_warp_ok(const NpadCommon2& cm, bool herm, bool trows) {
  if (trows || !herm || cm.inT != nullptr || cm.n > kMaxN) return false;
  const char* d = getenv("QCH_NPAD_DRIVER");
  return d == nullptr || strcmp(d, "block") != 0;
}

int npad_launch_full_warp(NpadJob2* jobs, int njobs, const NpadCommon2& cm, cudaStream_t st) {
  const size_t smem = sizeof(double2) * (size_t)cm.n * kPitch;
  auto kern = cm.stats ? (cm.ek ? npad_full_warp_kernel<true, true> : npad_full_warp_kernel<false, true>)
                       : (cm.ek ? npad_full_warp_kernel<true, false> : npad_full_warp_kernel<false, false>);
  QCH_CUDA(smem_attr((const void*)kern, (int)(sizeof(double2) * kMaxN * kPitch)));
  void* pr = prof_begin("npad_run_kernel", st);
  kern<<<njobs, 32, smem, st>>>(jobs, cm);
  prof_end(pr, st);
  QCH_LAUNCH_CHECK("npad_full_warp_kernel");
  note_launch(1);
  return QCH_OK;
}

}  // namespace qch
