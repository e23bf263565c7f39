// npad_tsmem.cu — subspace-mode NPAD (npad_run with a small target set,
// npad.py:300-354) for up to one chain per SM, with the |T| target rows
// resident in SHARED memory: the low-latency driver for the tail of a sweep
// (BASELINE config 4) and for the per-GPU shards of a multi-GPU sweep.
//
// Why: a sweep's makespan is its longest chain (717 rotations at config 4)
// times the latency of one rotation, and the many-chain drivers spend that
// latency in dependent global round trips (row t, row u, T-row rescans).
// Every rotation of subspace mode pairs a target row t (in T) with a partner
// u (not in T), and only T-rows carry candidates (npad.py:307-310).  Keeping
// the |T| x N T-rows in shared memory (eager: every entry always current)
// leaves ONE global round trip per rotation — the partner row u — and makes
// the T-row rescans shared-memory scans.
//
// Storage.  T-rows: shared memory, authoritative for every entry (t, x) and,
// by bitwise Hermiticity, (x, t).  Non-T rows: global, row-authoritative with
// clocks ("lazy columns", npad_cta.cu): entry (u, x), x not in T, lives in
// whichever of rows u, x was rotated later.  When the chain stops, the
// T-rows, their columns and the lazy columns of the rotated partner rows are
// written back, so the matrix in memory equals the eagerly updated one bit
// for bit (the arithmetic is npad_cta.cu's, statement for statement).
#include <algorithm>
#include <cstdlib>

#include "npad_run.h"
#include "npad_select.cuh"
#include "qch_internal.h"

namespace qch {
namespace {

constexpr int kTsThreads = 256;
constexpr int kTsWarps = kTsThreads / 32;

__device__ __forceinline__ bool below_thr_s(const Cand& p, double thr, bool ek) {
  if (ek) return p.q < thr;
  const double t2 = thr * thr;
  if (p.q > t2 * (1.0 + kRel)) return false;
  if (p.q < t2 * (1.0 - kRel)) return true;
  return np_cabs_ool(p.v.x, p.v.y) < thr;
}
// candidate for the relevant pair {t, x}: the lower-triangle entry H[max, min]
__device__ __forceinline__ Cand tcand_s(double2 htx, int t, int x, bool ek) {
  const bool tl = t > x;
  const double2 v = tl ? htx : make_double2(htx.x, -htx.y);
  const unsigned cr = tl ? (((unsigned)x << 16) | (unsigned)t) : (((unsigned)t << 16) | (unsigned)x);
  return make_cand(v, cr, ek);
}
__device__ __forceinline__ int partner_s(unsigned cr, int t) {
  const int c = (int)(cr >> 16), r = (int)(cr & 0xffffu);
  return c == t ? r : c;
}
__device__ __forceinline__ Cand shfl_cand_s(const Cand& c, int src) {
  Cand o;
  o.q = __shfl_sync(kFull, c.q, src);
  o.m = __shfl_sync(kFull, c.m, src);
  o.cr = __shfl_sync(kFull, c.cr, src);
  o.v.x = __shfl_sync(kFull, c.v.x, src);
  o.v.y = __shfl_sync(kFull, c.v.y, src);
  return o;
}
__device__ __forceinline__ double2 conj2s(double2 v) { return make_double2(v.x, -v.y); }

// running best of one row's candidates in increasing column order (ties keep
// the smaller column), exact numpy magnitudes inside the certification band
struct RowBestS {
  double hi, lo;
  int x;
  double2 v;
};
__device__ __forceinline__ void rbs_init(RowBestS& b) {
  b.hi = 0.0;
  b.lo = 1.0e308;
  b.x = -1;
  b.v = make_double2(0.0, 0.0);
}
__device__ __noinline__ bool mag_greater_s(double2 a, double2 b) { return np_cabs(a.x, a.y) > np_cabs(b.x, b.y); }
__device__ __forceinline__ void rbs_take(RowBestS& b, double2 v, int x) {
  const double q = fma(v.x, v.x, v.y * v.y);
  if (q > b.hi || (q >= b.lo && mag_greater_s(v, b.v))) {
    b.hi = q * (1.0 + kRel);
    b.lo = q * (1.0 - kRel);
    b.x = x;
    b.v = v;
  }
}

// rotate_rows with real-by-complex products as two rounded multiplies (as
// npad_cta.cu: numpy's (c + 0j) * z gives the same values for finite z)
__device__ __forceinline__ void rotate_rows_s(double c, cplx s, cplx ri, cplx rj, cplx* ni, cplx* nj) {
  const cplx b = np_cmul(cconj(s), rj);
  *ni = mkc(QSUB(QMUL(c, ri.re), b.re), QSUB(QMUL(c, ri.im), b.im));
  const cplx d = np_cmul(s, ri);
  *nj = mkc(QADD(d.re, QMUL(c, rj.re)), QADD(d.im, QMUL(c, rj.im)));
}

// block-wide best (every thread gets it); contains a barrier
__device__ __forceinline__ Cand block_best_s(Cand c, Cand* s_part, int lane, int warp) {
  const int wl = warp_argmax(c);
  const Cand w = (wl >= 0) ? shfl_cand_s(c, wl) : cand_none();
  if (lane == 0) s_part[warp] = w;
  __syncthreads();
  Cand b = s_part[0];
#pragma unroll
  for (int k = 1; k < kTsWarps; ++k) cand_take(b, s_part[k]);
  return b;
}

template <bool EK, bool ST>  // ST: per-phase cycle counters (QCH_NPAD_STATS), compiled out otherwise
__global__ void __launch_bounds__(kTsThreads, 1) npad_tsmem_kernel(NpadJob2* __restrict__ jobs, NpadCommon2 cm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = cm.n, nT = cm.n_target;
  constexpr bool ek = EK;
  extern __shared__ __align__(16) unsigned char smem[];
  double2* sT = (double2*)smem;                                     // [nT][n] target rows
  double* s_dg = (double*)(sT + (size_t)nT * n);                    // [n] diagonal (real)
  int* s_clk = (int*)(s_dg + n);                                    // [n] last rotation of a non-T row
  int* s_kof = s_clk + n;                                           // [n] index in T, -1 outside
  Cand* s_part = (Cand*)(((uintptr_t)(s_kof + n) + 15) & ~(uintptr_t)15);  // [kTsWarps]
  int* s_list = (int*)(s_part + kTsWarps);                          // [n] rotated rows (final pass)
  __shared__ int s_cnt;

  NpadJob2* job = jobs + blockIdx.x;
  double2* __restrict__ h = job->h;
  if (job->status == 0 || job->status == 1) return;  // finished in an earlier phase (2: paused, 3: fresh)
  for (int x = tid; x < n; x += kTsThreads) {
    s_clk[x] = 0;
    s_kof[x] = -1;
    s_dg[x] = h[(size_t)x * n + x].x;
  }
  __syncthreads();
  for (int k = tid; k < nT; k += kTsThreads) s_kof[cm.tlist[k]] = k;
  for (int k = 0; k < nT; ++k) {
    const double2* row = h + (size_t)cm.tlist[k] * n;
    for (int x = tid; x < n; x += kTsThreads) sT[(size_t)k * n + x] = row[x];
  }
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

  long long cyc[5] = {0, 0, 0, 0, 0};  // QCH_NPAD_STATS: select, row u + rotate, block best, fold, rescans
  while (true) {
    const long long c0 = ST ? clock64() : 0;
    // ---- selection (every warp, identical result)
    const int pl = warp_argmax(mine);
    Cand piv = cand_none();
    if (pl >= 0) piv = shfl_cand_s(mine, pl);
    if (applied >= cm.stop_at) {
      status = 2;
      break;
    }
    if (!(piv.q > 0.0) || below_thr_s(piv, thr, ek)) {
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
        __ballot_sync(kFull, lane < nT && lane != kt && (mine.q > 0.0) && partner_s(mine.cr, my_t) == u);
    const int wu = s_clk[u];
    double2* __restrict__ hu_r = h + (size_t)u * n;
    double2* __restrict__ sTt = sT + (size_t)kt * n;
    if (tid == 0 && pivots != nullptr && applied < pivot_cap) {
      pivots[2 * applied] = i;
      pivots[2 * applied + 1] = j;
    }
    const long long c1 = ST ? clock64() : 0;
    // ---- the partner row u: the ONE global round trip (all loads in flight)
    constexpr int kMaxCpt = 8;  // n <= 2048
    double2 ru[kMaxCpt];
    unsigned sm = 0u;
#pragma unroll
    for (int k = 0; k < kMaxCpt; ++k) {
      const int x = k * kTsThreads + tid;
      if (x < n) {
        const int kx = s_kof[x];
        if (kx >= 0) {
          ru[k] = conj2s(sT[(size_t)kx * n + u]);  // T-rows are authoritative
        } else {
          const bool a = s_clk[x] > wu;
          sm |= (a ? 1u : 0u) << k;
          ru[k] = a ? h[(size_t)x * n + u] : hu_r[x];
        }
      }
    }
    const double hii = s_dg[i], hjj = s_dg[j];
    const cplx v = d2c(piv.v);
    double c;
    cplx s;
    givens_fast(v, hii, hjj, &c, &s);  // rotation scalars (npad.py:101-128)
    RowBestS lbt;
    rbs_init(lbt);
    Cand pt = cand_none();
#pragma unroll
    for (int k = 0; k < kMaxCpt; ++k) {
      const int x = k * kTsThreads + tid;
      if (x >= n) break;
      const double2 vu = ((sm >> k) & 1u) ? conj2s(ru[k]) : ru[k];
      const double2 vt = sTt[x];
      cplx ni, nj;
      if (t_is_i) rotate_rows_s(c, s, d2c(vt), d2c(vu), &ni, &nj);
      else rotate_rows_s(c, s, d2c(vu), d2c(vt), &ni, &nj);
      const double2 nt = c2d(t_is_i ? ni : nj), nu = c2d(t_is_i ? nj : ni);
      sTt[x] = nt;  // columns t, u get provisional values; the 2x2 block overwrites them
      hu_r[x] = nu;
      const int kx = s_kof[x];
      if (kx < 0) {
        if (x != u) {
          if (EK) cand_take(pt, tcand_s(nt, t, x, ek));
          else rbs_take(lbt, nt, x);
        }
      } else if (x != t) {  // another T-row: its columns t and u changed (bitwise Hermitian)
        sT[(size_t)kx * n + t] = conj2s(nt);
        sT[(size_t)kx * n + u] = conj2s(nu);
      }
    }
    if (!EK && lbt.x >= 0) pt = tcand_s(lbt.v, t, lbt.x, ek);
    // the 2x2 block (npad.py:136-144 incl. the Hermitian pin); its coupling
    // H[j, i] is a candidate of T-row t
    const Block2 blk = rotate_block(c, s, mkc(hii, 0.0), cconj(v), v, mkc(hjj, 0.0));
    if (tid == 0) cand_take(pt, make_cand(c2d(blk.ji), ((unsigned)i << 16) | (unsigned)j, ek));
    const long long c2 = ST ? clock64() : 0;
    const Cand bt = block_best_s(pt, s_part, lane, warp);  // barrier: rows and folds visible
    const long long c3 = ST ? clock64() : 0;
    ++clock;
    if (tid == 0) {
      const double2 bii = c2d(blk.ii), bij = c2d(blk.ij), bji = c2d(blk.ji), bjj = c2d(blk.jj);
      sTt[t] = t_is_i ? bii : bjj;
      sTt[u] = t_is_i ? bij : bji;
      hu_r[u] = t_is_i ? bjj : bii;
      hu_r[t] = t_is_i ? bji : bij;
      s_dg[i] = blk.ii.re;
      s_dg[j] = blk.jj.re;
      s_clk[u] = clock;
    }
    if (lane == kt) mine = bt;
    // fold column u into the other T-rows; a T-row whose argmax partner was u
    // keeps it when the new entry is not smaller, otherwise it is rescanned
    bool need = false;
    if (lane < nT && lane != kt) {
      const Cand f = tcand_s(sT[(size_t)lane * n + u], my_t, u, ek);
      if ((resc >> lane) & 1u) {
        if (!cand_better(mine, f)) mine = f;
        else need = true;
      } else {
        cand_take(mine, f);
      }
    }
    unsigned rm = __ballot_sync(kFull, need);
    __syncthreads();  // 2x2 block, diagonal and clocks visible; s_part reusable
    const long long c4 = ST ? clock64() : 0;
    // ---- rescans of T-rows: shared memory only
    while (rm) {
      const int kr = __ffs(rm) - 1;
      rm &= rm - 1;
      ++rescans;
      const int tr = cm.tlist[kr];
      const double2* row = sT + (size_t)kr * n;
      RowBestS lbr;
      rbs_init(lbr);
      Cand pr = cand_none();
      for (int x = tid; x < n; x += kTsThreads) {
        if (s_kof[x] >= 0) continue;
        if (EK) cand_take(pr, tcand_s(row[x], tr, x, ek));
        else rbs_take(lbr, row[x], x);
      }
      if (!EK && lbr.x >= 0) pr = tcand_s(lbr.v, tr, lbr.x, ek);
      const Cand br = block_best_s(pr, s_part, lane, warp);
      if (lane == kr) mine = br;
      __syncthreads();  // s_part reuse
    }
    if (ST) {
      const long long c5 = clock64();
      cyc[0] += c1 - c0;
      cyc[1] += c2 - c1;
      cyc[2] += c3 - c2;
      cyc[3] += c4 - c3;
      cyc[4] += c5 - c4;
    }
    ++applied;
  }
  if (ST && tid == 0 && applied > 0)
    printf("npad tsmem driver: chain %d: %lld rotations, %.2f rescans/rot, cycles/rot: select %.0f, row u + rotate "
           "%.0f, block best %.0f, fold %.0f, rescans %.0f\n",
           blockIdx.x, applied, (double)rescans / applied, (double)cyc[0] / applied, (double)cyc[1] / applied,
           (double)cyc[2] / applied, (double)cyc[3] / applied, (double)cyc[4] / applied);

  // ---- write back: T-rows and their columns, then the lazy columns of the
  // rotated partner rows where they are the newer copy
  for (int k = 0; k < nT; ++k) {
    const int t = cm.tlist[k];
    double2* row = h + (size_t)t * n;
    const double2* srow = sT + (size_t)k * n;
    for (int x = tid; x < n; x += kTsThreads) {
      const double2 val = srow[x];
      row[x] = val;
      if (s_kof[x] < 0) h[(size_t)x * n + t] = conj2s(val);
    }
  }
  if (tid == 0) s_cnt = 0;
  __syncthreads();
  for (int x = tid; x < n; x += kTsThreads)
    if (s_clk[x] > 0) s_list[atomicAdd(&s_cnt, 1)] = x;
  __syncthreads();
  const int cnt = s_cnt;
  for (int q = 0; q < cnt; ++q) {
    const int y = s_list[q];
    const int wy = s_clk[y];
    const double2* __restrict__ row = h + (size_t)y * n;
    for (int x = tid; x < n; x += kTsThreads)
      if (x != y && s_kof[x] < 0 && s_clk[x] < wy) h[(size_t)x * n + y] = conj2s(row[x]);
  }
  if (lane < nT && warp == 0) {
    job->st_q[lane] = mine.q;
    job->st_c[lane] = (int)mine.cr;
    job->st_v[lane] = mine.v;
  }
  if (tid == 0) {
    job->applied = applied;
    job->status = status;
    if (ST) job->stats[0] += rescans;
  }
}

size_t tsmem_bytes(int n, int nT) {
  return (size_t)16 * nT * n + (size_t)8 * n + (size_t)4 * n + (size_t)4 * n + 16 + sizeof(Cand) * kTsWarps +
         (size_t)4 * n;
}

}  // namespace

// shared memory needed for one chain (0 when the driver does not apply)
size_t npad_tsmem_bytes(const NpadCommon2& cm) {
  if (cm.n_target < 1 || cm.n_target > 32 || cm.n > 8 * kTsThreads) return 0;
  const size_t b = tsmem_bytes(cm.n, cm.n_target);
  return b <= (size_t)max_smem_optin() ? b : 0;
}

int npad_launch_tsmem(NpadJob2* jobs, int njobs, const NpadCommon2& cm, cudaStream_t st) {
  const size_t smem = npad_tsmem_bytes(cm);
  if (smem == 0) return fail(QCH_ERR_UNSUPPORTED, "npad: shared-memory T-rows driver does not fit");
  auto kern = cm.stats ? (cm.ek ? npad_tsmem_kernel<true, true> : npad_tsmem_kernel<false, true>)
                       : (cm.ek ? npad_tsmem_kernel<true, false> : npad_tsmem_kernel<false, false>);
  QCH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  void* pr = prof_begin("npad_run_kernel", st);
  kern<<<njobs, kTsThreads, smem, st>>>(jobs, cm);
  prof_end(pr, st);
  QCH_LAUNCH_CHECK("npad_tsmem_kernel");
  note_launch(1);
  return QCH_OK;
}

}  // namespace qch
