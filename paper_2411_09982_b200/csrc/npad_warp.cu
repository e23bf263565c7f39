// npad_warp.cu — subspace-mode NPAD (npad_run with a small target set,
// npad.py:300-354) with ONE WARP per greedy chain: the parameter-sweep
// driver (BASELINE config 4: 1024 independent dim-1024 chains).
//
// Why a warp: a chain is a serial sequence of rotations.  One warp per chain
// keeps block barriers off the critical path (shuffles only), makes all 1024
// chains resident at once (~7 per SM) and lets their memory traffic overlap:
// the sweep becomes bandwidth-bound instead of latency-bound.
//
// Algorithm (identical pivots to the reference; see npad_run.cu "T-rows"):
// the relevant couplings of subspace mode are H[t, x], t in T, x not in T
// (npad.py:307-310).  Lane l < |T| keeps the best candidate of T-row l (key
// desc, then the reference's (i, j) tie-break, npad_select.cuh).
//
// Row-authoritative storage ("lazy columns").  A rotation (t, u) changes rows
// AND columns t, u; the reference writes both (npad.py:136-144).  Writing the
// two columns costs 2N scattered 16-byte stores (each a 32-byte DRAM
// read-modify-write) — three quarters of the DRAM traffic of the eager
// kernel.  Here only ROWS are written during the chain.  Every row carries
// the clock of its last rotation (rows never rotated: 0); the true entry
// (x, y) lives in whichever of rows x, y was rotated last (the matrix is
// bitwise Hermitian, so entry (x, y) = conj(entry (y, x)) of that row).  When
// a row is read (rotation inputs, T-row rescans), its entries at the few
// columns y whose rows were rotated later ("stale" columns: the chain touches
// only ~40 distinct rows) are patched with conj(H[y, x]).  When the chain
// stops, one fix-up pass writes the columns of the touched rows, so the
// matrix in memory is exactly the eager result (same bits).
//
// Streaming: rows are pulled through a 4-stage cp.async ring of 128-column
// stages (up to 16 KB in flight per chain; the stale-column gathers ride in
// the first group), patched in shared memory, rotated with the reference's
// arithmetic (qch_math.cuh), written back coalesced.  The new row t is
// reduced on the fly; column u's new entries H[t', u] are folded into the
// other T-rows via shared memory; a T-row whose stored argmax partner was u
// keeps it when the new entry did not shrink, and is otherwise rescanned
// (whole row in one cp.async pass).
#include <algorithm>
#include <cstdlib>

#include "npad_run.h"
#include "npad_select.cuh"
#include "qch_internal.h"

namespace qch {

constexpr int kStageCols = 128;  // columns per stage (4 per lane)
constexpr int kStages = 4;       // ring depth
constexpr int kTouchCap = 128;   // distinct touched rows tracked before a flush
constexpr int kStaleCap = 128;   // stale columns per row read (bounded by kTouchCap)

__device__ __forceinline__ bool below_thr_w(const Cand& p, double thr, bool ek) {
  // mag < threshold with mag the exact numpy |z| (npad.py:348)
  if (ek) return p.q < thr;
  const double t2 = thr * thr;
  if (p.q > t2 * (1.0 + kRel)) return false;
  if (p.q < t2 * (1.0 - kRel)) return true;
  return np_cabs_ool(p.v.x, p.v.y) < thr;
}

// candidate for the relevant pair {t, x}: the lower-triangle entry H[max, min]
__device__ __forceinline__ Cand tcand(double2 htx, int t, int x, bool ek) {
  const bool tl = t > x;
  const double2 v = tl ? htx : make_double2(htx.x, -htx.y);
  const unsigned cr = tl ? (((unsigned)x << 16) | (unsigned)t) : (((unsigned)t << 16) | (unsigned)x);
  return make_cand(v, cr, ek);
}
__device__ __forceinline__ int partner(unsigned cr, int t) {
  const int c = (int)(cr >> 16), r = (int)(cr & 0xffffu);
  return c == t ? r : c;
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

// Per-lane running best of a row's candidates H[t, x] over the lane's
// columns, visited in increasing x.  For a fixed row t the reference's
// tie-break (magnitude desc, then lower-triangle (c, r) asc) is simply x asc,
// so a strictly larger key replaces the best; keys within the certification
// band (npad_select.cuh) are resolved with exact numpy magnitudes, equal ones
// keep the earlier (smaller) x.
struct LaneBest {
  double hi, lo;  // certified band of the current best key
  int x;
  double2 v;      // H[t, x]
};
__device__ __forceinline__ void lb_init(LaneBest& b) {
  b.hi = 0.0;
  b.lo = 1.0e308;
  b.x = -1;
  b.v = make_double2(0.0, 0.0);
}
static __device__ __noinline__ bool mag_greater(double2 a, double2 b) {
  return np_cabs(a.x, a.y) > np_cabs(b.x, b.y);
}
__device__ __forceinline__ void lb_take(LaneBest& b, double2 v, int x) {
  const double q = fma(v.x, v.x, v.y * v.y);
  if (q > b.hi) {
    b.hi = q * (1.0 + kRel);
    b.lo = q * (1.0 - kRel);
    b.x = x;
    b.v = v;
  } else if (q >= b.lo && mag_greater(v, b.v)) {
    b.hi = q * (1.0 + kRel);
    b.lo = q * (1.0 - kRel);
    b.x = x;
    b.v = v;
  }
}

// rotate_rows (qch_math.cuh, npad.py:136-137) with the real-by-complex
// products as two rounded multiplies: numpy's (c + 0j) * z gives the same
// values for finite z (up to the sign of an exact zero), in 16 instead of 24
// FP64 instructions
__device__ __forceinline__ void rotate_rows_fast(double c, cplx s, cplx ri, cplx rj, cplx* ni, cplx* nj) {
  const cplx b = np_cmul(cconj(s), rj);
  *ni = mkc(QSUB(QMUL(c, ri.re), b.re), QSUB(QMUL(c, ri.im), b.im));
  const cplx d = np_cmul(s, ri);
  *nj = mkc(QADD(d.re, QMUL(c, rj.re)), QADD(d.im, QMUL(c, rj.im)));
}

__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ double2 conj2(double2 v) { return make_double2(v.x, -v.y); }
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int W>
__device__ __forceinline__ void cpa_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(W) : "memory");
}

// per-warp shared-memory layout
struct WarpSm {
  double2 ring[kStages][2][kStageCols];  // 16 KB
  double2 diag[2];
  double2 fold[32];
  double2 stale_v[2][kStaleCap];
  int stale_c[2][kStaleCap];
  int touch_row[kTouchCap];
  int touch_w[kTouchCap];
};

// per-chain touched-row bookkeeping (warp-uniform values; list in shared)
struct Touch {
  WarpSm* sm;
  unsigned* bits;  // n bits: row touched since the last flush
  int count;
};

// clock of row r's last rotation (0: never, since the last flush)
__device__ __forceinline__ int row_clock(const Touch& tc, int r, int lane) {
  if (!((tc.bits[r >> 5] >> (r & 31)) & 1u)) return 0;
  int w = 0;
  for (int k = lane; k < tc.count; k += 32)
    if (tc.sm->touch_row[k] == r) w = tc.sm->touch_w[k];
  return __reduce_max_sync(kFull, w);
}

// columns of row r that are stale (their row was rotated after row r): the
// list goes to stale_c[slot]; the raw entries H[y, r] are fetched with
// cp.async into stale_v[slot] (their conjugates are the true H[r, y]; the
// caller commits the group).  Returns the count (warp-uniform).
__device__ __forceinline__ int gather_stale(const Touch& tc, const double2* __restrict__ h, int n, int r, int wr,
                                            int slot, int lane) {
  int cnt = 0;
  for (int base = 0; base < tc.count; base += 32) {
    const int k = base + lane;
    const bool st = k < tc.count && tc.sm->touch_w[k] > wr;
    const unsigned m = __ballot_sync(kFull, st);
    if (st) {
      const int pos = cnt + __popc(m & ((1u << lane) - 1u));
      const int y = tc.sm->touch_row[k];
      tc.sm->stale_c[slot][pos] = y;
      cpa16(&tc.sm->stale_v[slot][pos], h + (size_t)y * n + r);
    }
    cnt += __popc(m);
  }
  return cnt;
}
// write the columns of every touched row where that row is the newer one:
// afterwards the matrix in memory is exactly the eagerly updated one
__device__ void flush_columns(Touch& tc, double2* __restrict__ h, int n, int lane) {
  double2* flat = &tc.sm->ring[0][0][0];
  constexpr int kFlat = kStages * 2 * kStageCols;
  for (int k = 0; k < tc.count; ++k) {
    const int y = tc.sm->touch_row[k];
    const int wy = tc.sm->touch_w[k];
    const double2* __restrict__ row = h + (size_t)y * n;
    for (int base = 0; base < n; base += kFlat) {
      const int cnt = min(kFlat, n - base);
      for (int q = lane; q < cnt; q += 32) cpa16(flat + q, row + base + q);
      cpa_commit();
      cpa_wait<0>();
      __syncwarp();
      for (int q = lane; q < cnt; q += 32) {
        const int x = base + q;
        if (x == y) continue;
        int wx = 0;
        if ((tc.bits[x >> 5] >> (x & 31)) & 1u) {
          for (int p = 0; p < tc.count; ++p)
            if (tc.sm->touch_row[p] == x) wx = tc.sm->touch_w[p];
        }
        if (wx < wy) h[(size_t)x * n + y] = conj2(flat[q]);
      }
      __syncwarp();
    }
  }
  __syncwarp();
  for (int k = lane; k < tc.count; k += 32) {
    const int y = tc.sm->touch_row[k];
    atomicAnd(&tc.bits[y >> 5], ~(1u << (y & 31)));
  }
  tc.count = 0;
  __syncwarp();
}

// record row r as rotated at clock w (the caller guarantees room)
__device__ __forceinline__ void touch(Touch& tc, int r, int w, int lane) {
  const bool had = (tc.bits[r >> 5] >> (r & 31)) & 1u;
  if (had) {
    for (int k = lane; k < tc.count; k += 32)
      if (tc.sm->touch_row[k] == r) tc.sm->touch_w[k] = w;
  } else {
    if (lane == 0) {
      tc.sm->touch_row[tc.count] = r;
      tc.sm->touch_w[tc.count] = w;
      tc.bits[r >> 5] |= 1u << (r & 31);
    }
    ++tc.count;
  }
  __syncwarp();
}

// EK: exact keys (q := numpy |z|) for matrices whose entries could leave the
// normal range of |z|^2 (npad.cu:exact_keys) — the generic candidate path.
template <bool EK, bool FULL, bool ST>  // ST: per-phase cycle counters (QCH_NPAD_STATS), compiled out otherwise
__global__ void __launch_bounds__(256, 1) npad_trows_warp_kernel(NpadJob2* __restrict__ jobs, int njobs,
                                                              NpadCommon2 cm) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int n = cm.n, nT = cm.n_target;
  constexpr bool ek = EK;
  const int nwords = (n + 31) / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  WarpSm* wsm = (WarpSm*)smem + wib;
  int* s_kof = (int*)(smem + sizeof(WarpSm) * wpb);  // x -> index in T, -1 outside (block-shared)
  unsigned* s_bits = (unsigned*)(s_kof + n) + (size_t)wib * nwords;

  for (int x = threadIdx.x; x < n; x += blockDim.x) s_kof[x] = -1;
  __syncthreads();
  for (int k = threadIdx.x; k < nT; k += blockDim.x) s_kof[cm.tlist[k]] = k;
  __syncthreads();

  const int jb = blockIdx.x * wpb + wib;
  if (jb >= njobs) return;
  NpadJob2* job = jobs + jb;
  double2* __restrict__ h = job->h;
  for (int k = lane; k < nwords; k += 32) s_bits[k] = 0u;
  // T membership of this lane's columns x = 32 k + lane (n <= 1024: a register)
  // FULL: n is a multiple of the stage width and <= 1024, so each lane's
  // columns are x = 32 k + lane, k < 32: T membership fits a register
  const bool small_n = FULL;
  unsigned tmask = 0u;
  if (small_n)
    for (int k = 0; k * 32 + lane < n; ++k)
      if (s_kof[k * 32 + lane] >= 0) tmask |= 1u << k;
  Touch tc{wsm, s_bits, 0};
  Cand mine = cand_none();  // lane l: T-row l
  int my_t = -1;
  if (lane < nT) {
    my_t = cm.tlist[lane];
    mine.q = job->st_q[lane];
    mine.m = -1.0;
    mine.cr = (unsigned)job->st_c[lane];
    mine.v = job->st_v[lane];
  }
  __syncwarp();
  auto in_T = [&](int x) -> bool { return small_n ? ((tmask >> (x >> 5)) & 1u) != 0u : s_kof[x] >= 0; };

  long long applied = job->applied;
  const double thr = job->threshold;
  int* const pivots = job->pivots;
  const long long pivot_cap = job->pivot_cap;
  int status = 0;
  long long rescans = 0;
  int clock = 0;
  const int nstage = (n + kStageCols - 1) / kStageCols;

  long long cyc_sel = 0, cyc_stage = 0, cyc_post = 0;
  while (true) {
    const long long c0 = ST ? clock64() : 0;
    // ---- selection over the |T| T-row candidates
    Cand sel = mine;
    const int pl = warp_argmax(sel);
    if (pl >= 0 && lane < nT) mine.m = sel.m;  // keep a computed exact magnitude
    Cand piv = cand_none();
    if (pl >= 0) piv = shfl_cand(sel, pl);
    if (applied >= cm.stop_at) {
      status = 2;
      break;
    }
    if (!(piv.q > 0.0) || below_thr_w(piv, thr, ek)) {
      status = 0;
      break;
    }
    if (applied >= cm.max_iter) {
      status = 1;
      break;
    }
    // hand the chain over to the low-latency driver once few chains are left
    if (cm.live != nullptr && (applied & 15) == 0 && *(volatile int*)cm.live <= cm.handover) {
      status = 2;
      break;
    }
    const int i = (int)(piv.cr >> 16), j = (int)(piv.cr & 0xffffu);
    const int t = s_kof[i] >= 0 ? i : j;
    const int kt = s_kof[t];
    const int u = (t == i) ? j : i;
    const bool t_is_i = (t == i);
    const unsigned resc = __ballot_sync(kFull, lane < nT && lane != kt && (mine.q > 0.0) && partner(mine.cr, my_t) == u);
    const double2* __restrict__ ri_p = h + (size_t)i * n;
    const double2* __restrict__ rj_p = h + (size_t)j * n;
    // room for two new touched rows: flush BEFORE reading rows i, j (the
    // matrix is then fully consistent and nothing is stale)
    if (tc.count + 2 > kTouchCap) flush_columns(tc, h, n, lane);

    const long long c1 = ST ? clock64() : 0;
    // ---- stale lists + their async gathers and the two diagonal entries
    // (rows own their diagonal: never stale) ride in the first commit group
    // with ring stage 0; the ring streams rows i, j
    const int wi = row_clock(tc, i, lane), wj = row_clock(tc, j, lane);
    const int ns_i = gather_stale(tc, h, n, i, wi, 0, lane);
    const int ns_j = gather_stale(tc, h, n, j, wj, 1, lane);
    if (lane == 0) cpa16(&wsm->diag[0], ri_p + i);
    if (lane == 1) cpa16(&wsm->diag[1], rj_p + j);
    // per-lane addresses of the ring (shared) and of rows i, j (global)
    const unsigned ring_sa = (unsigned)__cvta_generic_to_shared(&wsm->ring[0][0][lane]);
    const double2* __restrict__ ri_l = ri_p + lane;
    const double2* __restrict__ rj_l = rj_p + lane;
    auto issue = [&](int stg) {
      if (stg < nstage) {
        const unsigned sa = ring_sa + (unsigned)((stg & (kStages - 1)) * 2 * kStageCols * 16);
        const int base = stg * kStageCols;
#pragma unroll
        for (int k = 0; k < kStageCols / 32; ++k) {
          if (FULL || base + k * 32 + lane < n) {
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa + k * 32 * 16), "l"(ri_l + base + k * 32)
                         : "memory");
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa + (kStageCols + k * 32) * 16),
                         "l"(rj_l + base + k * 32)
                         : "memory");
          }
        }
      }
      cpa_commit();
    };
#pragma unroll
    for (int stg = 0; stg < kStages - 1; ++stg) issue(stg);
    if (lane == 0 && pivots != nullptr && applied < pivot_cap) {
      pivots[2 * applied] = i;
      pivots[2 * applied + 1] = j;
    }
    const cplx v = d2c(piv.v);
    double c = 0.0, hii = 0.0, hjj = 0.0;
    cplx s = mkc(0.0, 0.0);

    LaneBest lbt;  // new row t (fast keys)
    lb_init(lbt);
    Cand pt = cand_none();  // new row t (exact keys)
#pragma unroll 1
    for (int stg = 0; stg < nstage; ++stg) {
      issue(stg + kStages - 1);
      cpa_wait<kStages - 1>();
      __syncwarp();
      if (stg == 0) {
        // rotation scalars (every lane, same values): givens_rotation_matrix
        // + _block_params (npad.py:101-128)
        hii = wsm->diag[0].x;
        hjj = wsm->diag[1].x;
        givens_fast(v, hii, hjj, &c, &s);
      }
      const int slot = stg & (kStages - 1);
      const int base = stg * kStageCols;
      // patch stale columns of this stage
      if (ns_i + ns_j > 0) {
        for (int q = lane; q < ns_i; q += 32) {
          const int y = wsm->stale_c[0][q];
          if (y >= base && y < base + kStageCols) wsm->ring[slot][0][y - base] = conj2(wsm->stale_v[0][q]);
        }
        for (int q = lane; q < ns_j; q += 32) {
          const int y = wsm->stale_c[1][q];
          if (y >= base && y < base + kStageCols) wsm->ring[slot][1][y - base] = conj2(wsm->stale_v[1][q]);
        }
        __syncwarp();
      }
      // rotate this stage.  Columns i, j get provisional values here; the 2x2
      // block below overwrites them (same warp, after a __syncwarp).
      const double2* __restrict__ ra = &wsm->ring[slot][0][lane];
      const double2* __restrict__ rb = &wsm->ring[slot][1][lane];
      double2* __restrict__ oi = h + (size_t)i * n + base + lane;
      double2* __restrict__ oj = h + (size_t)j * n + base + lane;
      const bool full = FULL || base + kStageCols <= n;
      const unsigned tbits = FULL ? (tmask >> (base >> 5)) : 0u;
#pragma unroll
      for (int k = 0; k < kStageCols / 32; ++k) {
        const int x = base + k * 32 + lane;
        if (!full && x >= n) break;
        cplx ni, nj;
        rotate_rows_fast(c, s, d2c(ra[k * 32]), d2c(rb[k * 32]), &ni, &nj);
        oi[k * 32] = c2d(ni);
        oj[k * 32] = c2d(nj);
        const bool inTx = FULL ? ((tbits >> k) & 1u) != 0u : s_kof[x] >= 0;
        if (!inTx) {
          if (x != u) {
            if (EK) {
              cand_take(pt, tcand(c2d(t_is_i ? ni : nj), t, x, ek));
            } else {
              lb_take(lbt, c2d(t_is_i ? ni : nj), x);
            }
          }
        } else if (x != t) {
          // x = t' in T: new H[t', u] = conj(new H[u, t'])
          wsm->fold[s_kof[x]] = c2d(cconj(t_is_i ? nj : ni));
        }
      }
      __syncwarp();  // ring slot reuse
    }
    cpa_wait<0>();
    const long long c2 = ST ? clock64() : 0;
    __syncwarp();  // provisional writes of columns i, j before the 2x2 block
    if (!EK && lbt.x >= 0) pt = tcand(lbt.v, t, lbt.x, ek);
    // the 2x2 block (npad.py:136-144 incl. the Hermitian pin) and its
    // coupling H[j, i] as a candidate of T-row t
    if (lane == 0) {
      const Block2 b = rotate_block(c, s, mkc(hii, 0.0), cconj(v), v, mkc(hjj, 0.0));
      h[(size_t)i * n + i] = c2d(b.ii);
      h[(size_t)i * n + j] = c2d(b.ij);
      h[(size_t)j * n + i] = c2d(b.ji);
      h[(size_t)j * n + j] = c2d(b.jj);
      cand_take(pt, make_cand(c2d(b.ji), ((unsigned)i << 16) | (unsigned)j, ek));
    }
    ++clock;
    touch(tc, i, clock, lane);
    touch(tc, j, clock, lane);
    __syncwarp();  // row writes and fold visible to the warp
    {
      const int wl = warp_argmax(pt);
      const Cand best = (wl >= 0) ? shfl_cand(pt, wl) : cand_none();
      if (lane == kt) mine = best;
    }
    // fold column u into the other T-rows.  A T-row whose argmax partner was u
    // keeps it if the new entry is not smaller; otherwise it is rescanned.
    unsigned rm = 0;
    {
      bool need = false;
      if (lane < nT && lane != kt) {
        Cand f = tcand(wsm->fold[lane], my_t, u, ek);
        if ((resc >> lane) & 1u) {
          if (!cand_better(mine, f)) {
            mine = f;  // still the largest entry of its row
          } else {
            need = true;
          }
        } else {
          cand_take(mine, f);
        }
      }
      rm = __ballot_sync(kFull, need);
    }
    // rescans: the whole row in one shot through the ring (1024 columns per
    // pass), stale columns patched from gathers
    while (rm) {
      const int kr = __ffs(rm) - 1;
      rm &= rm - 1;
      ++rescans;
      const int tr = cm.tlist[kr];
      const int wt = row_clock(tc, tr, lane);
      const int ns = gather_stale(tc, h, n, tr, wt, 0, lane);
      const double2* __restrict__ row = h + (size_t)tr * n;
      double2* flat = &wsm->ring[0][0][0];
      constexpr int kFlat = kStages * 2 * kStageCols;
      Cand pr = cand_none();
      LaneBest lbr;
      lb_init(lbr);
      for (int base = 0; base < n; base += kFlat) {
        const int cnt = min(kFlat, n - base);
        for (int q = lane; q < cnt; q += 32) cpa16(flat + q, row + base + q);
        cpa_commit();
        cpa_wait<0>();
        __syncwarp();
        for (int q = lane; q < ns; q += 32) {
          const int y = wsm->stale_c[0][q];
          if (y >= base && y < base + cnt) flat[y - base] = conj2(wsm->stale_v[0][q]);
        }
        __syncwarp();
        for (int q = lane; q < cnt; q += 32) {
          const int x = base + q;
          if (in_T(x)) continue;
          if (EK) {
            cand_take(pr, tcand(flat[q], tr, x, ek));
          } else {
            lb_take(lbr, flat[q], x);
          }
        }
        __syncwarp();
      }
      if (!EK && lbr.x >= 0) pr = tcand(lbr.v, tr, lbr.x, ek);
      const int wl = warp_argmax(pr);
      const Cand best = (wl >= 0) ? shfl_cand(pr, wl) : cand_none();
      if (lane == kr) mine = best;
    }
    if (ST) {
      const long long c3 = clock64();
      cyc_sel += c1 - c0;
      cyc_stage += c2 - c1;
      cyc_post += c3 - c2;
    }
    ++applied;
  }

  flush_columns(tc, h, n, lane);  // the matrix in memory is the eager result again
  if (lane < nT) {
    job->st_q[lane] = mine.q;
    job->st_c[lane] = (int)mine.cr;
    job->st_v[lane] = mine.v;
  }
  if (lane == 0) {
    job->applied = applied;
    job->status = status;
    if (cm.live != nullptr && status != 2) atomicSub(cm.live, 1);
    if (ST) {
      job->stats[0] += rescans;
      job->stats[1] += cyc_sel;
      job->stats[2] += cyc_stage;
      job->stats[3] += cyc_post;
      if (blockIdx.x == 0 && wib == 0)
        printf("npad warp driver: chain 0: %lld rotations, %.2f rescans/rot, cycles/rot: select %.0f, rows %.0f, "
               "fold+rescan %.0f\n", applied, (double)rescans / (applied ? applied : 1),
               (double)cyc_sel / (applied ? applied : 1), (double)cyc_stage / (applied ? applied : 1),
               (double)cyc_post / (applied ? applied : 1));
    }
  }
}

size_t trows_warp_smem(int n, int wpb) {
  return sizeof(WarpSm) * wpb + (size_t)4 * n + (size_t)4 * ((n + 31) / 32) * wpb;
}

int npad_launch_trows_warp(NpadJob2* jobs, int njobs, const NpadCommon2& cm, cudaStream_t st) {
  // ~3+ blocks per SM so the chains spread evenly over the SMs
  int wpb = 8;
  while (wpb > 1 && ((int64_t)njobs + wpb - 1) / wpb < 3 * sm_count()) wpb >>= 1;
  if (const char* e = getenv("QCH_NPAD_WPB")) wpb = std::max(1, std::min(8, atoi(e)));
  while (wpb > 1 && trows_warp_smem(cm.n, wpb) > (size_t)max_smem_optin()) wpb >>= 1;
  const size_t smem = trows_warp_smem(cm.n, wpb);
  if (smem > (size_t)max_smem_optin()) return fail(QCH_ERR_UNSUPPORTED, "npad: warp T-rows driver shared memory");
  const bool full = cm.n % kStageCols == 0 && cm.n <= 1024;
  auto kern = cm.stats
                  ? (cm.ek ? (full ? npad_trows_warp_kernel<true, true, true> : npad_trows_warp_kernel<true, false, true>)
                           : (full ? npad_trows_warp_kernel<false, true, true> : npad_trows_warp_kernel<false, false, true>))
                  : (cm.ek ? (full ? npad_trows_warp_kernel<true, true, false> : npad_trows_warp_kernel<true, false, false>)
                           : (full ? npad_trows_warp_kernel<false, true, false>
                                   : npad_trows_warp_kernel<false, false, false>));
  QCH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = (njobs + wpb - 1) / wpb;
  void* pr = prof_begin("npad_run_kernel", st);
  kern<<<grid, 32 * wpb, smem, st>>>(jobs, njobs, cm);
  prof_end(pr, st);
  QCH_LAUNCH_CHECK("npad_trows_warp_kernel");
  note_launch(1);
  return QCH_OK;
}

}  // namespace qch
