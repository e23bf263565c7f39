// npad_cta.cu — subspace-mode NPAD (npad_run with a small target set,
// npad.py:300-354) for MANY independent chains: the parameter-sweep driver
// (BASELINE config 4: 1024 dim-1024 chains), one 128-thread CTA per chain.
//
// A chain is a serial sequence of rotations, so the sweep's run time is set
// by its longest chain (717 rotations here) times the latency of one
// rotation — not by aggregate throughput.  A 128-thread CTA splits each row
// 8 columns per thread: a rotation is ONE memory round trip (every thread
// issues all its loads at once) plus two block barriers.  (npad_warp.cu is the
// one-warp-per-chain variant: cheaper per chain, longer per rotation.)
//
// Algorithm (identical pivots to the reference; see npad_run.cu "T-rows"):
// the relevant couplings of subspace mode are H[t, x], t in T, x not in T
// (npad.py:307-310).  Every warp keeps the |T| T-row candidates redundantly
// (lane l: T-row l; key desc, then the reference's (i, j) tie-break,
// npad_select.cuh) and applies identical updates, so the pivot needs no
// broadcast.
//
// Row-authoritative storage ("lazy columns").  A rotation (t, u) changes rows
// AND columns t, u; the reference writes both (npad.py:136-144).  Writing the
// two columns costs 2N scattered 16-byte stores (each a 32-byte DRAM
// read-modify-write) — three quarters of the DRAM traffic of an eager update.
// Here only ROWS are written.  Each row has a clock (shared memory) = the
// rotation that last wrote it (0: never); the true entry (x, y) is in
// whichever of rows x, y is newer (bitwise Hermitian: entry (x, y) =
// conj(entry (y, x)) of that row).  A thread reading H[r, x] therefore loads
// conj(H[x, r]) instead when clock[x] > clock[r] — same single load, other
// address, no extra round trip.  When the chain stops, one pass writes the
// columns of the rotated rows (only ~40 distinct rows per sweep chain), so
// the matrix in memory is exactly the eagerly updated one, bit for bit.
#include <algorithm>
#include <cstdlib>

#include "npad_run.h"
#include "npad_select.cuh"
#include "qch_internal.h"

namespace qch {
namespace {

constexpr int kCtaThreads = 128;  // threads per chain
constexpr int kCtaWarps = kCtaThreads / 32;
constexpr int kCpt = 8;           // columns per thread per pass (one pass = 1024 columns)

__device__ __forceinline__ bool below_thr_c(const Cand& p, double thr, bool ek) {
  // mag < threshold with mag the exact numpy |z| (npad.py:348)
  if (ek) return p.q < thr;
  const double t2 = thr * thr;
  if (p.q > t2 * (1.0 + kRel)) return false;
  if (p.q < t2 * (1.0 - kRel)) return true;
  return np_cabs_ool(p.v.x, p.v.y) < thr;
}

// candidate for the relevant pair {t, x}: the lower-triangle entry H[max, min]
__device__ __forceinline__ Cand tcand_c(double2 htx, int t, int x, bool ek) {
  const bool tl = t > x;
  const double2 v = tl ? htx : make_double2(htx.x, -htx.y);
  const unsigned cr = tl ? (((unsigned)x << 16) | (unsigned)t) : (((unsigned)t << 16) | (unsigned)x);
  return make_cand(v, cr, ek);
}
__device__ __forceinline__ int partner_c(unsigned cr, int t) {
  const int c = (int)(cr >> 16), r = (int)(cr & 0xffffu);
  return c == t ? r : c;
}
__device__ __forceinline__ Cand shfl_cand_c(const Cand& c, int src) {
  Cand o;
  o.q = __shfl_sync(kFull, c.q, src);
  o.m = __shfl_sync(kFull, c.m, src);
  o.cr = __shfl_sync(kFull, c.cr, src);
  o.v.x = __shfl_sync(kFull, c.v.x, src);
  o.v.y = __shfl_sync(kFull, c.v.y, src);
  return o;
}
__device__ __forceinline__ double2 conj2c(double2 v) { return make_double2(v.x, -v.y); }

// Per-thread running best of row t's candidates H[t, x] over the thread's
// columns, visited in increasing x.  For a fixed row the reference's
// tie-break (magnitude desc, then lower-triangle (c, r) asc) is x asc, so a
// strictly larger key replaces the best; keys within the certification band
// (npad_select.cuh) are resolved with exact numpy magnitudes.
struct RowBest {
  double hi, lo;
  int x;
  double2 v;
};
__device__ __forceinline__ void rb_init(RowBest& b) {
  b.hi = 0.0;
  b.lo = 1.0e308;
  b.x = -1;
  b.v = make_double2(0.0, 0.0);
}
__device__ __noinline__ bool mag_greater_c(double2 a, double2 b) { return np_cabs(a.x, a.y) > np_cabs(b.x, b.y); }
__device__ __forceinline__ void rb_take(RowBest& b, double2 v, int x) {
  const double q = fma(v.x, v.x, v.y * v.y);
  if (q > b.hi || (q >= b.lo && mag_greater_c(v, b.v))) {
    b.hi = q * (1.0 + kRel);
    b.lo = q * (1.0 - kRel);
    b.x = x;
    b.v = v;
  }
}

// rotate_rows (qch_math.cuh, npad.py:136-137) with the real-by-complex
// products as two rounded multiplies: numpy's (c + 0j) * z gives the same
// values for finite z (up to the sign of an exact zero)
__device__ __forceinline__ void rotate_rows_c(double c, cplx s, cplx ri, cplx rj, cplx* ni, cplx* nj) {
  const cplx b = np_cmul(cconj(s), rj);
  *ni = mkc(QSUB(QMUL(c, ri.re), b.re), QSUB(QMUL(c, ri.im), b.im));
  const cplx d = np_cmul(s, ri);
  *nj = mkc(QADD(d.re, QMUL(c, rj.re)), QADD(d.im, QMUL(c, rj.im)));
}

// block-wide best of the per-thread candidates (every thread gets it);
// contains the barrier that publishes everything written before it
__device__ __forceinline__ Cand block_best(Cand c, Cand* s_part, int lane, int warp) {
  const int wl = warp_argmax(c);
  const Cand w = (wl >= 0) ? shfl_cand_c(c, wl) : cand_none();
  if (lane == 0) s_part[warp] = w;
  __syncthreads();
  Cand b = s_part[0];
#pragma unroll
  for (int k = 1; k < kCtaWarps; ++k) cand_take(b, s_part[k]);
  return b;
}

template <bool EK>
__global__ void __launch_bounds__(kCtaThreads, 4) npad_trows_cta_kernel(NpadJob2* __restrict__ jobs, NpadCommon2 cm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = cm.n, nT = cm.n_target;
  constexpr bool ek = EK;
  extern __shared__ __align__(16) unsigned char smem[];
  int* s_clk = (int*)smem;  // per-row clock of the last rotation (0: never)
  int* s_kof = s_clk + n;   // x -> index in T, -1 outside
  double2* s_fold = (double2*)(smem + (((size_t)8 * n + 15) & ~(size_t)15));  // [32] new H[t', u]
  Cand* s_part = (Cand*)(s_fold + 32);                                          // [kCtaWarps]
  int* s_list = (int*)(s_part + kCtaWarps);                                    // rotated rows (final pass)
  __shared__ int s_cnt;

  NpadJob2* job = jobs + blockIdx.x;
  double2* __restrict__ h = job->h;
  for (int x = tid; x < n; x += kCtaThreads) {
    s_clk[x] = 0;
    s_kof[x] = -1;
  }
  __syncthreads();
  for (int k = tid; k < nT; k += kCtaThreads) s_kof[cm.tlist[k]] = k;
  Cand mine = cand_none();  // lane l (every warp): T-row l
  int my_t = -1;
  if (lane < nT) {
    my_t = cm.tlist[lane];
    mine.q = job->st_q[lane];
    mine.m = -1.0;
    mine.cr = (unsigned)job->st_c[lane];
    mine.v = job->st_v[lane];
  }
  __syncthreads();

  long long applied = job->applied;
  const double thr = job->threshold;
  int* const pivots = job->pivots;
  const long long pivot_cap = job->pivot_cap;
  int status = 0;
  long long rescans = 0;
  int clock = 0;
  const int npass = (n + kCtaThreads * kCpt - 1) / (kCtaThreads * kCpt);

  while (true) {
    // ---- selection (every warp, identical result)
    Cand sel = mine;
    const int pl = warp_argmax(sel);
    Cand piv = cand_none();
    if (pl >= 0) piv = shfl_cand_c(sel, pl);
    if (applied >= cm.stop_at) {
      status = 2;
      break;
    }
    if (!(piv.q > 0.0) || below_thr_c(piv, thr, ek)) {
      status = 0;
      break;
    }
    if (applied >= cm.max_iter) {
      status = 1;
      break;
    }
    const int i = (int)(piv.cr >> 16), j = (int)(piv.cr & 0xffffu);
    const int t = s_kof[i] >= 0 ? i : j;
    const int kt = s_kof[t];
    const int u = (t == i) ? j : i;
    const bool t_is_i = (t == i);
    const unsigned resc =
        __ballot_sync(kFull, lane < nT && lane != kt && (mine.q > 0.0) && partner_c(mine.cr, my_t) == u);
    const int wi = s_clk[i], wj = s_clk[j];
    double2* __restrict__ hi_r = h + (size_t)i * n;
    double2* __restrict__ hj_r = h + (size_t)j * n;
    if (tid == 0 && pivots != nullptr && applied < pivot_cap) {
      pivots[2 * applied] = i;
      pivots[2 * applied + 1] = j;
    }
    const double hii = hi_r[i].x, hjj = hj_r[j].x;  // rows own their diagonal (never stale)
    const cplx v = d2c(piv.v);
    double c = 0.0;
    cplx s = mkc(0.0, 0.0);
    RowBest lbt;
    rb_init(lbt);
    Cand pt = cand_none();
#pragma unroll 1
    for (int pass = 0; pass < npass; ++pass) {
      // ---- one round trip: every load of this pass in flight at once; a
      // stale entry is read from its newer mirror, conj(H[x, r])
      double2 ra[kCpt], rb[kCpt];
      unsigned sm = 0u;
#pragma unroll
      for (int k = 0; k < kCpt; ++k) {
        const int x = (pass * kCpt + k) * kCtaThreads + tid;
        if (x < n) {
          const int cx = s_clk[x];
          const bool a = cx > wi, b = cx > wj;
          sm |= (a ? 1u : 0u) << (2 * k);
          sm |= (b ? 2u : 0u) << (2 * k);
          ra[k] = a ? h[(size_t)x * n + i] : hi_r[x];
          rb[k] = b ? h[(size_t)x * n + j] : hj_r[x];
        }
      }
      if (pass == 0) givens_fast(v, hii, hjj, &c, &s);  // rotation scalars (npad.py:101-128)
#pragma unroll
      for (int k = 0; k < kCpt; ++k) {
        const int x = (pass * kCpt + k) * kCtaThreads + tid;
        if (x >= n) break;
        const double2 va = ((sm >> (2 * k)) & 1u) ? conj2c(ra[k]) : ra[k];
        const double2 vb = ((sm >> (2 * k)) & 2u) ? conj2c(rb[k]) : rb[k];
        cplx ni, nj;
        rotate_rows_c(c, s, d2c(va), d2c(vb), &ni, &nj);
        hi_r[x] = c2d(ni);  // columns i, j get provisional values; the 2x2 block overwrites them
        hj_r[x] = c2d(nj);
        const int kx = s_kof[x];
        if (kx < 0) {
          if (x != u) {
            if (EK) {
              cand_take(pt, tcand_c(c2d(t_is_i ? ni : nj), t, x, ek));
            } else {
              rb_take(lbt, c2d(t_is_i ? ni : nj), x);
            }
          }
        } else if (x != t) {
          s_fold[kx] = c2d(cconj(t_is_i ? nj : ni));  // new H[t', u] = conj(new H[u, t'])
        }
      }
    }
    if (!EK && lbt.x >= 0) pt = tcand_c(lbt.v, t, lbt.x, ek);
    // the 2x2 block (npad.py:136-144 incl. the Hermitian pin); its coupling
    // H[j, i] is a candidate of T-row t
    const Block2 blk = rotate_block(c, s, mkc(hii, 0.0), cconj(v), v, mkc(hjj, 0.0));
    if (tid == 0) cand_take(pt, make_cand(c2d(blk.ji), ((unsigned)i << 16) | (unsigned)j, ek));
    const Cand bt = block_best(pt, s_part, lane, warp);  // barrier: rows, fold, partials visible
    ++clock;
    if (tid == 0) {
      hi_r[i] = c2d(blk.ii);
      hi_r[j] = c2d(blk.ij);
      hj_r[i] = c2d(blk.ji);
      hj_r[j] = c2d(blk.jj);
      s_clk[i] = clock;
      s_clk[j] = clock;
    }
    if (lane == kt) mine = bt;
    // fold column u into the other T-rows; a T-row whose argmax partner was u
    // keeps it when the new entry is not smaller, otherwise it is rescanned
    bool need = false;
    if (lane < nT && lane != kt) {
      const Cand f = tcand_c(s_fold[lane], my_t, u, ek);
      if ((resc >> lane) & 1u) {
        if (!cand_better(mine, f)) mine = f;
        else need = true;
      } else {
        cand_take(mine, f);
      }
    }
    unsigned rm = __ballot_sync(kFull, need);
    __syncthreads();  // 2x2 block + clocks visible; s_part / s_fold reusable
    // ---- rescans of T-rows (whole row, one round trip per pass)
    while (rm) {
      const int kr = __ffs(rm) - 1;
      rm &= rm - 1;
      ++rescans;
      const int tr = cm.tlist[kr];
      const int wt = s_clk[tr];
      const double2* __restrict__ row = h + (size_t)tr * n;
      RowBest lbr;
      rb_init(lbr);
      Cand pr = cand_none();
#pragma unroll 1
      for (int pass = 0; pass < npass; ++pass) {
        double2 ra[kCpt];
        unsigned sm = 0u;
#pragma unroll
        for (int k = 0; k < kCpt; ++k) {
          const int x = (pass * kCpt + k) * kCtaThreads + tid;
          if (x < n) {
            const bool a = s_clk[x] > wt;
            sm |= (a ? 1u : 0u) << k;
            ra[k] = a ? h[(size_t)x * n + tr] : row[x];
          }
        }
#pragma unroll
        for (int k = 0; k < kCpt; ++k) {
          const int x = (pass * kCpt + k) * kCtaThreads + tid;
          if (x >= n) break;
          if (s_kof[x] >= 0) continue;
          const double2 val = ((sm >> k) & 1u) ? conj2c(ra[k]) : ra[k];
          if (EK) {
            cand_take(pr, tcand_c(val, tr, x, ek));
          } else {
            rb_take(lbr, val, x);
          }
        }
      }
      if (!EK && lbr.x >= 0) pr = tcand_c(lbr.v, tr, lbr.x, ek);
      const Cand br = block_best(pr, s_part, lane, warp);
      if (lane == kr) mine = br;
      __syncthreads();  // s_part reuse
    }
    ++applied;
  }

  // ---- write the columns of the rotated rows where they are the newer copy
  if (tid == 0) s_cnt = 0;
  __syncthreads();
  for (int x = tid; x < n; x += kCtaThreads)
    if (s_clk[x] > 0) s_list[atomicAdd(&s_cnt, 1)] = x;
  __syncthreads();
  const int cnt = s_cnt;
  for (int q = 0; q < cnt; ++q) {
    const int y = s_list[q];
    const int wy = s_clk[y];
    const double2* __restrict__ row = h + (size_t)y * n;
    for (int x = tid; x < n; x += kCtaThreads)
      if (x != y && s_clk[x] < wy) h[(size_t)x * n + y] = conj2c(row[x]);
  }
  if (lane < nT && warp == 0) {
    job->st_q[lane] = mine.q;
    job->st_c[lane] = (int)mine.cr;
    job->st_v[lane] = mine.v;
  }
  if (tid == 0) {
    job->applied = applied;
    job->status = status;
    if (cm.stats) job->stats[0] += rescans;
  }
}

size_t trows_cta_smem(int n) {
  return (((size_t)8 * n + 15) & ~(size_t)15) + sizeof(double2) * 32 + sizeof(Cand) * kCtaWarps + (size_t)4 * n;
}

}  // namespace

int npad_launch_trows_cta(NpadJob2* jobs, int njobs, const NpadCommon2& cm, cudaStream_t st) {
  const size_t smem = trows_cta_smem(cm.n);
  if (smem > (size_t)max_smem_optin()) return fail(QCH_ERR_UNSUPPORTED, "npad: CTA T-rows driver shared memory");
  auto kern = cm.ek ? npad_trows_cta_kernel<true> : npad_trows_cta_kernel<false>;
  QCH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  void* pr = prof_begin("npad_run_kernel", st);
  kern<<<njobs, kCtaThreads, smem, st>>>(jobs, cm);
  prof_end(pr, st);
  QCH_LAUNCH_CHECK("npad_trows_cta_kernel");
  note_launch(1);
  return QCH_OK;
}

}  // namespace qch
