// npad_coop.cu — ONE greedy NPAD chain (npad_run, npad.py:320-354) spread
// over the whole GPU: the full-diagonal driver for large dense operators
// (BASELINE config 3: dim 4096, 292,068 rotations).
//
// A single chain is serial (each pick needs the previous rotation), and one
// SM cannot move the ~400 KB a dim-4096 rotation touches in less than tens
// of microseconds.  Here G CTAs (one per SM, cooperative launch) share the
// chain.  CTA g owns a contiguous block of ROWS R_g (their incremental
// best-candidate state, in shared memory) and the same block of COLUMNS
// C_g = R_g.  Per rotation (i, j):
//
//   phase A (every CTA, no communication)
//     * rotate rows i, j on the columns x in C_g (npad.py:136-137), write
//       them and the mirrored columns H[x, i], H[x, j] (the matrix stays
//       bitwise Hermitian, npad.py:139-144) — those are rows x in R_g;
//     * fold the two new entries of each own row x into its best candidate;
//       rows whose best sat in column i or j are rescanned by the CTA;
//     * partial bests of the NEW rows i and j over C_g (the 2x2 block's
//       H[j, i] included by the owner of column i), and the best over the own
//       rows other than i, j; published to a double-buffered record array;
//   publish (release), then wait for every CTA's record (acquire);
//   phase B (every CTA redundantly, identical results)
//     * combine the G partials into the new row-i / row-j candidates (their
//       owners store them) and pick the global pivot with the reference
//       order (npad_select.cuh: certified |z|^2 keys, numpy |z| near ties,
//       (mag desc, i asc, j asc));
//     * every CTA keeps a full copy of the diagonal and updates it from the
//       2x2 block it computes itself, so the rotation scalars need no load.
//
// The records carry the rotation count as an epoch (release store after the
// CTA's matrix writes); waiting for all G records of an epoch (acquire) IS the
// grid barrier — one per rotation, no atomics.  Bit-identical to the
// single-CTA driver (same arithmetic, same candidate order).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "npad_run.h"
#include "npad_select.cuh"
#include "qch_internal.h"

namespace qch {
namespace {

constexpr int kCoopThreads = 256;
constexpr int kMaxCoopCtas = 1024;  // stats buffer rows (G <= SM count)
constexpr int kCoopWarps = kCoopThreads / 32;
constexpr int kRescanBatch = 16;  // loads in flight per thread in a row rescan (a dim-4096 row in one batch)

struct CoopRec {
  Cand own;   // best over the CTA's rows other than i, j
  Cand pi;    // new row i over the CTA's columns
  Cand pj;    // new row j over the CTA's columns
  int epoch;  // = rotations applied when published (release store; readers acquire)
};

struct CoopArgs {
  double2* h;
  double2* u;          // nullable: accumulated unitary, rows i, j updated (npad.py:244-251)
  int n;
  int rows_per;        // rows (and columns) per CTA
  int ek;
  double threshold;
  long long max_iter;
  const double* st_q;  // initial row state (rows_init_kernel)
  const int* st_c;
  const double2* st_v;
  CoopRec* rec;        // [2][G]; epochs initialised to -1
  int* pivots;
  long long pivot_cap;
  long long* out_applied;
  int* out_status;
  long long* stats;  // non-null (QCH_NPAD_STATS): CTA 0 phase cycles [wait, combine, scalars, rotate, rescan, publish], rescans
  int mbx;           // cluster mode: records by st.async onto byte-counting mbarriers (else barrier.cluster)
  int pf_rescan;     // bulk-prefetch the rows about to be rescanned into L2 when the pivot is known
};

// one 16-byte piece of a record field into a peer CTA's shared memory, its
// bytes counted on the peer's mbarrier (st.async: the completion has release
// semantics at cluster scope)
__device__ __forceinline__ void st_async16(unsigned raddr, unsigned rbar, const void* src) {
  const unsigned long long* p = (const unsigned long long*)src;
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "l"(p[0]), "l"(p[1]), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned map_rank(unsigned addr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// wait for a phase of a local mbarrier; acquire at cluster scope (the peers'
// matrix writes ordered before their records become visible)
__device__ __forceinline__ void mbar_wait_cluster(unsigned bar, unsigned par) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
          bar),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void mbar_arm(unsigned bar, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
}
// a Cand field (48 bytes) of this CTA's record into peer `rank`
__device__ __forceinline__ void send_cand(const Cand& c, Cand* local_field, unsigned local_bar, unsigned rank) {
  static_assert(sizeof(Cand) == 48, "Cand layout");
  const unsigned ra = map_rank(smem_addr(local_field), rank), rb = map_rank(local_bar, rank);
  const unsigned char* src = (const unsigned char*)&c;
#pragma unroll
  for (int k = 0; k < 3; ++k) st_async16(ra + 16 * k, rb, src + 16 * k);
}

__device__ __forceinline__ int ld_acq(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_rel(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ Cand shfl_cand_p(const Cand& c, int src) {
  Cand o;
  o.q = __shfl_sync(kFull, c.q, src);
  o.m = __shfl_sync(kFull, c.m, src);
  o.cr = __shfl_sync(kFull, c.cr, src);
  o.v.x = __shfl_sync(kFull, c.v.x, src);
  o.v.y = __shfl_sync(kFull, c.v.y, src);
  return o;
}
__device__ __forceinline__ Cand warp_best(Cand c) {
  const int wl = warp_argmax(c);
  return (wl >= 0) ? shfl_cand_p(c, wl) : cand_none();
}

// T independent warp argmaxes with their REDUX / ballot steps interleaved
// (the same winners as T warp_best calls; the rare near-tie path stays exact)
template <int T>
__device__ __forceinline__ void warp_best_n(Cand* const (&cs)[T]) {
  unsigned long long bb[T];
  unsigned hh[T], hm[T], lm[T], nb[T];
  bool nf[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    bb[t] = (cs[t]->q > 0.0) ? (unsigned long long)__double_as_longlong(cs[t]->q) : 0ull;
    hh[t] = (unsigned)(bb[t] >> 32);
  }
#pragma unroll
  for (int t = 0; t < T; ++t) hm[t] = __reduce_max_sync(kFull, hh[t]);
#pragma unroll
  for (int t = 0; t < T; ++t) lm[t] = __reduce_max_sync(kFull, (hh[t] == hm[t]) ? (unsigned)bb[t] : 0u);
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const double qs = __longlong_as_double((long long)(((unsigned long long)hm[t] << 32) | lm[t]));
    nf[t] = (cs[t]->q > 0.0) && (cs[t]->q >= qs * (1.0 - kRel));
  }
#pragma unroll
  for (int t = 0; t < T; ++t) nb[t] = __ballot_sync(kFull, nf[t]);
  int w[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    w[t] = -1;
    if (hm[t] != 0u)
      w[t] = (__popc(nb[t]) == 1) ? __ffs(nb[t]) - 1 : warp_argmax_exact(cs[t]->v, cs[t]->m, cs[t]->cr, nf[t]);
  }
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const Cand o = shfl_cand_p(*cs[t], w[t] >= 0 ? w[t] : 0);
    *cs[t] = w[t] >= 0 ? o : cand_none();
  }
}
// three block-wide bests at once for the publish step, where only warp 0
// (the record writers) needs them: per-warp bests, then warp 0 reduces the
// kCoopWarps partials of each with a warp argmax — one barrier, no broadcast;
// s_part: 3 * kCoopWarps entries
__device__ __forceinline__ void block_best3_w0(Cand& a, Cand& b, Cand& c, Cand* s_part) {
  const Cand wa = warp_best(a), wb = warp_best(b), wc = warp_best(c);
  const int w = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  if (lane == 0) {
    s_part[w] = wa;
    s_part[kCoopWarps + w] = wb;
    s_part[2 * kCoopWarps + w] = wc;
  }
  __syncthreads();
  if (w == 0) {
    Cand x = lane < kCoopWarps ? s_part[lane] : cand_none();
    Cand y = lane < kCoopWarps ? s_part[kCoopWarps + lane] : cand_none();
    Cand z = lane < kCoopWarps ? s_part[2 * kCoopWarps + lane] : cand_none();
    a = warp_best(x);
    b = warp_best(y);
    c = warp_best(z);
  }
}
// block-wide best (every thread gets it); s_part: kCoopWarps entries
__device__ __forceinline__ Cand block_best_p(const Cand& c, Cand* s_part) {
  const Cand w = warp_best(c);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = w;
  __syncthreads();
  Cand b = s_part[0];
#pragma unroll
  for (int k = 1; k < kCoopWarps; ++k) cand_take(b, s_part[k]);
  __syncthreads();
  return b;
}

constexpr int kClusterMax = 16;

// CL: the G CTAs form ONE thread-block cluster; records travel through
// distributed shared memory (each CTA writes its record into every CTA's
// s_rec) and the per-rotation barrier is barrier.cluster (release/acquire at
// cluster scope, which also orders the CTAs' global matrix writes) instead of
// polling epoch-flagged records in global memory.
template <bool EK, bool CL, bool ST>  // ST: per-phase cycle counters (QCH_NPAD_STATS)
__global__ void __launch_bounds__(kCoopThreads, 1) npad_coop_kernel(const __grid_constant__ CoopArgs a) {
  namespace cg = cooperative_groups;
  __shared__ CoopRec s_rec[CL ? 2 : 1][CL ? kClusterMax : 1];
  __shared__ __align__(8) unsigned long long s_xbar[2];  // CL + mbx: record bytes of a publication
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp_u = __shfl_sync(0xffffffffu, tid >> 5, 0);  // provably warp-uniform (converged shuffles)
  const int G = gridDim.x, g = blockIdx.x;
  const int n = a.n;
  constexpr bool ek = EK;
  const int r0 = g * a.rows_per, r1 = min(n, r0 + a.rows_per);
  const int nr = max(0, r1 - r0);
  extern __shared__ __align__(16) unsigned char smem[];
  double* s_dg = (double*)smem;                  // full diagonal copy
  Cand* s_row = (Cand*)(smem + (((size_t)8 * n + 15) & ~(size_t)15));  // best candidate of each own row
  Cand* s_part = s_row + a.rows_per;             // [kCoopWarps] reduction scratch
  Cand* s_rpart = s_part + 3 * kCoopWarps + 3;    // [2][kCoopWarps] rescan partials (double-buffered)
  int* s_resc = (int*)(s_rpart + 2 * kCoopWarps);  // own rows to rescan
  __shared__ int s_nresc;
  double2* __restrict__ h = a.h;

  for (int x = tid; x < n; x += kCoopThreads) s_dg[x] = h[(size_t)x * n + x].x;
  for (int k = tid; k < nr; k += kCoopThreads) {
    const int x = r0 + k;
    Cand c = cand_none();
    if (a.st_q[x] > 0.0) {
      c.q = a.st_q[x];
      c.cr = ((unsigned)a.st_c[x] << 16) | (unsigned)x;
      c.v = a.st_v[x];
    }
    s_row[k] = c;
  }
  __syncthreads();

  long long applied = 0;
  int status = 0;
  int pi_row = -1, pj_row = -1;  // rows whose state comes from the partials of the last rotation
  const bool mbx = CL && a.mbx != 0;
  const unsigned xtx = (unsigned)(G * 3 * sizeof(Cand));  // record bytes a CTA receives per publication
  if (mbx) {
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&s_xbar[0])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&s_xbar[1])) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_arm(smem_addr(&s_xbar[0]), xtx);
    }
    cg::this_cluster().sync();  // every CTA's barriers initialised before any record is sent
  }
  // first publication: own bests only
  {
    Cand own = cand_none();
    for (int k = tid; k < nr; k += kCoopThreads) cand_take(own, s_row[k]);
    own = block_best_p(own, s_part);
    if (mbx) {
      if (tid < G) {
        const Cand none = cand_none();
        const unsigned lb = smem_addr(&s_xbar[0]);
        send_cand(own, &s_rec[0][g].own, lb, tid);
        send_cand(none, &s_rec[0][g].pi, lb, tid);
        send_cand(none, &s_rec[0][g].pj, lb, tid);
      }
    } else if (CL) {
      if (tid < G) {
        CoopRec* r = cg::this_cluster().map_shared_rank(&s_rec[0][g], tid);
        r->own = own;
        r->pi = cand_none();
        r->pj = cand_none();
      }
      cg::this_cluster().sync();
    } else if (tid == 0) {
      a.rec[g].own = own;
      a.rec[g].pi = cand_none();
      a.rec[g].pj = cand_none();
      __threadfence();
      st_rel(&a.rec[g].epoch, 0);
    }
  }

  long long cyc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long ck = clock64();
  auto tick = [&](int k) {
    if (ST) {
      const long long c2 = clock64();
      cyc[k] += c2 - ck;
      ck = c2;
    }
  };
  while (true) {
    // ---- phase B: combine the records, pick the pivot (every CTA)
    // (waiting for every CTA's record of this epoch is the grid barrier: the
    // acquire makes each publisher's matrix writes visible)
    const CoopRec* rec = CL ? s_rec[applied & 1] : a.rec + (size_t)(applied & 1) * G;
    if (mbx) {
      mbar_wait_cluster(smem_addr(&s_xbar[applied & 1]), (unsigned)((applied >> 1) & 1));
      // the barrier of the next publication: its previous phase completed one rotation ago
      if (tid == 0) mbar_arm(smem_addr(&s_xbar[(applied + 1) & 1]), xtx);
    }
    if (!CL) {
      if (tid < 32) {
        for (int k = tid; k < G; k += 32)
          while (ld_acq(&a.rec[(size_t)(applied & 1) * G + k].epoch) != (int)applied) {
          }
      }
      __syncthreads();
    }
    tick(0);
    // global records: the G records are reduced by warp 0 alone (one
    // barrier; a block-wide reduction of at most G <= 148 records cost two
    // barriers and a serial cross-warp combine in every thread).  Cluster
    // (G <= 16 records in shared memory): every warp reduces them itself —
    // identical results, no barrier, no broadcast
    // The pivot is the best of ALL record entries (one warp argmax); the new
    // states of the last rotation's rows i, j (the combined pi / pj partials)
    // are reduced only by the CTAs that own those rows.
    const bool own_pi = pi_row >= r0 && pi_row < r1, own_pj = pj_row >= r0 && pj_row < r1;  // CTA-uniform
    Cand piv = cand_none(), cpi = cand_none(), cpj = cand_none();
    if (CL) {
      // every warp finds the pivot; the row-i / row-j states are reduced by
      // warps 1 and 2 of their owner CTAs, in parallel with the others
      const bool red_i = own_pi && warp_u == 1, red_j = own_pj && warp_u == 2;  // warp-uniform
      // G <= 16 records: lanes 0..15 fold own + pi of record `lane`, lanes
      // 16..31 pj of record `lane - 16` (two dependent folds per lane, not three)
      if (lane < G) {
        const Cand ro = rec[lane].own, rpi = rec[lane].pi;
        cand_take(piv, ro);
        cand_take(piv, rpi);
        if (red_i) cpi = rpi;
      } else if (lane >= 16 && lane - 16 < G) {
        const Cand rpj = rec[lane - 16].pj;
        cand_take(piv, rpj);
        if (red_j) cpj = rpj;
      }
      piv = warp_best(piv);
      if (red_i) {
        cpi = warp_best(cpi);
        if (lane == 0) s_row[pi_row - r0] = cpi;
      }
      if (red_j) {
        cpj = warp_best(cpj);
        if (lane == 0) s_row[pj_row - r0] = cpj;
      }
    } else {
      if (warp_u == 0) {
        for (int k = lane; k < G; k += 32) {
          const Cand ro = rec[k].own, rpi = rec[k].pi, rpj = rec[k].pj;
          cand_take(piv, ro);
          cand_take(piv, rpi);
          cand_take(piv, rpj);
          if (own_pi) cand_take(cpi, rpi);
          if (own_pj) cand_take(cpj, rpj);
        }
        piv = warp_best(piv);
        if (own_pi) cpi = warp_best(cpi);
        if (own_pj) cpj = warp_best(cpj);
        if (lane == 0) {
          s_part[0] = piv;
          if (own_pi) s_row[pi_row - r0] = cpi;
          if (own_pj) s_row[pj_row - r0] = cpj;
        }
      }
      __syncthreads();
      piv = s_part[0];
    }
    // (the new states of the last rotation's rows i, j are visible to the
    // rotation pass after the barrier below)
    if (!(piv.q > 0.0) || [&] {
          if (ek) return piv.q < a.threshold;
          const double t2 = a.threshold * a.threshold;
          if (piv.q > t2 * (1.0 + kRel)) return false;
          if (piv.q < t2 * (1.0 - kRel)) return true;
          return np_cabs(piv.v.x, piv.v.y) < a.threshold;
        }()) {
      status = 0;
      break;
    }
    if (applied >= a.max_iter) {
      status = 1;
      break;
    }
    tick(1);
    const int i = (int)(piv.cr >> 16), j = (int)(piv.cr & 0xffffu);
    // own rows whose best sat in column i or j will be rescanned after the
    // rotation: their lower-triangle entries start moving into L2 now (one
    // bulk prefetch per row), under the scalars and the rotation
    if (a.pf_rescan)
      for (int k = tid; k < nr; k += kCoopThreads) {
        const int bc = (int)(s_row[k].cr >> 16);  // (no candidate: cr = ~0 -> column 0xffff, never i or j)
        const int x = r0 + k;
        if ((bc == i || bc == j) && x != i && x != j && x > 0)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(h + (size_t)x * n),
                       "r"((unsigned)(x * sizeof(double2)))
                       : "memory");
      }
    if (g == 0 && tid == 0 && a.pivots != nullptr && applied < a.pivot_cap) {
      a.pivots[2 * applied] = i;
      a.pivots[2 * applied + 1] = j;
    }
    // this thread's first own column of rows i, j: issued before the scalars'
    // sqrt / rsqrt chain so the global loads overlap it
    double2 pre_i = make_double2(0.0, 0.0), pre_j = make_double2(0.0, 0.0);
    if (tid < nr) {
      pre_i = h[(size_t)i * n + r0 + tid];
      pre_j = h[(size_t)j * n + r0 + tid];
    }
    // rotation scalars and the 2x2 block: every thread, same values
    const cplx v = d2c(piv.v);
    const double hii = s_dg[i], hjj = s_dg[j];
    double c;
    cplx s;
    givens_fast(v, hii, hjj, &c, &s);
    const Block2 blk = rotate_block(c, s, mkc(hii, 0.0), cconj(v), v, mkc(hjj, 0.0));

    tick(2);
    // ---- phase A: own columns of rows i, j; mirrored columns = own rows
    if (tid == 0) s_nresc = 0;
    __syncthreads();
    Cand ppi = cand_none(), ppj = cand_none();
    // best over own rows other than i, j (their state arrives with the next
    // phase B), folded as each row's state is finalised: here, or by thread 0
    // after a rescan
    Cand own = cand_none();
    for (int k = tid; k < nr; k += kCoopThreads) {
      const int x = r0 + k;
      if (x == i || x == j) continue;
      const cplx ri = d2c(k == tid ? pre_i : h[(size_t)i * n + x]), rj = d2c(k == tid ? pre_j : h[(size_t)j * n + x]);
      cplx ni, nj;
      rotate_rows(c, s, ri, rj, &ni, &nj);
      h[(size_t)i * n + x] = c2d(ni);
      h[(size_t)j * n + x] = c2d(nj);
      h[(size_t)x * n + i] = c2d(cconj(ni));
      h[(size_t)x * n + j] = c2d(cconj(nj));
      // new rows i, j: lower-triangle entries (i, x) for x < i, (j, x) for x < j
      if (x < i) cand_take(ppi, make_cand(c2d(ni), ((unsigned)x << 16) | (unsigned)i, ek));
      if (x < j) cand_take(ppj, make_cand(c2d(nj), ((unsigned)x << 16) | (unsigned)j, ek));
      // own row x: its entries (x, i) if i < x and (x, j) if j < x changed
      Cand st = s_row[k];
      const int bc = (st.q > 0.0) ? (int)(st.cr >> 16) : -1;
      if (bc == i || bc == j) {
        s_resc[atomicAdd(&s_nresc, 1)] = x;
      } else {
        if (i < x) cand_take(st, make_cand(c2d(cconj(ni)), ((unsigned)i << 16) | (unsigned)x, ek));
        if (j < x) cand_take(st, make_cand(c2d(cconj(nj)), ((unsigned)j << 16) | (unsigned)x, ek));
        s_row[k] = st;
        cand_take(own, st);
      }
    }
    // accumulated unitary: rows i, j of U on the own columns (_apply_left,
    // npad.py:244-251; the same arithmetic as the single-CTA driver)
    if (a.u != nullptr) {
      double2* __restrict__ u = a.u;
      for (int x = r0 + tid; x < r1; x += kCoopThreads) {
        cplx ni, nj;
        rotate_rows(c, s, d2c(u[(size_t)i * n + x]), d2c(u[(size_t)j * n + x]), &ni, &nj);
        u[(size_t)i * n + x] = c2d(ni);
        u[(size_t)j * n + x] = c2d(nj);
      }
    }
    // the 2x2 block entries, by the owners of columns i and j
    if (tid == 0) {
      if (i >= r0 && i < r1) {
        h[(size_t)i * n + i] = c2d(blk.ii);
        h[(size_t)j * n + i] = c2d(blk.ji);
        cand_take(ppj, make_cand(c2d(blk.ji), ((unsigned)i << 16) | (unsigned)j, ek));
      }
      if (j >= r0 && j < r1) {
        h[(size_t)i * n + j] = c2d(blk.ij);
        h[(size_t)j * n + j] = c2d(blk.jj);
      }
    }
    s_dg[i] = blk.ii.re;  // every thread writes the same value
    s_dg[j] = blk.jj.re;
    __syncthreads();  // own rows' new entries written and visible to the CTA
    tick(3);
    // rescans of own rows whose best sat in column i or j (whole CTA per row)
    const int nresc = s_nresc;
    cyc[6] += nresc;
    for (int q = 0; q < nresc; ++q) {
      const int x = s_resc[q];
      const double2* __restrict__ row = h + (size_t)x * n;
      Cand b = cand_none();
      int bx = -1;
      double bhi = 0.0, blo = 1.0e308;
      double2 bv = make_double2(0.0, 0.0);
      for (int base = 0; base < x; base += kCoopThreads * kRescanBatch) {
        double2 vals[kRescanBatch];
#pragma unroll
        for (int k = 0; k < kRescanBatch; ++k) {
          const int cc = base + k * kCoopThreads + tid;
          vals[k] = cc < x ? row[cc] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int k = 0; k < kRescanBatch; ++k) {
          const int cc = base + k * kCoopThreads + tid;
          if (cc >= x) break;
          if (EK) {
            cand_take(b, make_cand(vals[k], ((unsigned)cc << 16) | (unsigned)x, ek));
          } else {
            // running best in increasing column order (ties keep the smaller column)
            const double qv = fma(vals[k].x, vals[k].x, vals[k].y * vals[k].y);
            if (qv > bhi || (qv >= blo && np_cabs_ool(vals[k].x, vals[k].y) > np_cabs_ool(bv.x, bv.y))) {
              bhi = qv * (1.0 + kRel);
              blo = qv * (1.0 - kRel);
              bx = cc;
              bv = vals[k];
            }
          }
        }
      }
      if (!EK && bx >= 0) b = make_cand(bv, ((unsigned)bx << 16) | (unsigned)x, ek);
      // block best: warp partials, then warp 0 alone (lane 0 writes the row
      // state).  The partials alternate between two buffers, so the next
      // row's partials never overwrite ones warp 0 may still be reading and
      // no trailing barrier is needed (the row state is read only after the
      // record exchange)
      Cand* rp = s_rpart + (q & 1) * kCoopWarps;
      b = warp_best(b);
      if (lane == 0) rp[tid >> 5] = b;
      __syncthreads();
      if (warp_u == 0) {
        Cand rb = lane < kCoopWarps ? rp[lane] : cand_none();
        rb = warp_best(rb);
        if (lane == 0) {
          s_row[x - r0] = rb;
          cand_take(own, rb);
        }
      }
    }
    tick(4);
    if (CL) {
      // per-warp bests, then warps 0, 1, 2 reduce own / pi / pj in parallel
      // and each writes its field of the record into every CTA
      Cand wa = own, wb = ppi, wc = ppj;
      {
        Cand* const cs3[3] = {&wa, &wb, &wc};
        warp_best_n<3>(cs3);
      }
      if (lane == 0) {
        s_part[warp_u] = wa;
        s_part[kCoopWarps + warp_u] = wb;
        s_part[2 * kCoopWarps + warp_u] = wc;
      }
      __syncthreads();
      tick(7);
      ++applied;
      if (warp_u < 3) {
        Cand x = lane < kCoopWarps ? s_part[warp_u * kCoopWarps + lane] : cand_none();
        x = warp_best(x);
        if (lane < G) {
          if (mbx) {
            CoopRec* lr = &s_rec[applied & 1][g];
            send_cand(x, warp_u == 0 ? &lr->own : warp_u == 1 ? &lr->pi : &lr->pj,
                      smem_addr(&s_xbar[applied & 1]), lane);
          } else {
            CoopRec* r = cg::this_cluster().map_shared_rank(&s_rec[applied & 1][g], lane);
            if (warp_u == 0)
              r->own = x;
            else if (warp_u == 1)
              r->pi = x;
            else
              r->pj = x;
          }
        }
      }
      // release/acquire: records and matrix writes (mbx: the records' st.async
      // completions release, the next phase B's wait acquires)
      if (!mbx) cg::this_cluster().sync();
    } else {
      block_best3_w0(own, ppi, ppj, s_part);  // valid in warp 0: the record writer
      tick(7);
      ++applied;
    }
    if (!CL && tid == 0) {
      CoopRec* w = a.rec + (size_t)(applied & 1) * G + g;
      w->own = own;
      w->pi = ppi;
      w->pj = ppj;
      __threadfence();
      st_rel(&w->epoch, (int)applied);
    }
    pi_row = i;
    pj_row = j;
    tick(5);
  }
  if (mbx) cg::this_cluster().sync();  // no CTA leaves while a peer may still address it
  if (ST && tid == 0)
    for (int k = 0; k < 8; ++k) a.stats[8 * g + k] = cyc[k];
  if (g == 0 && tid == 0) {
    *a.out_applied = applied;
    *a.out_status = status;
  }
}

}  // namespace

size_t npad_coop_smem(int n, int rows_per) {
  return (((size_t)8 * n + 15) & ~(size_t)15) + sizeof(Cand) * (rows_per + 5 * kCoopWarps + 3) + (size_t)4 * rows_per +
         64;
}

// Run the greedy full-diagonal chain of ONE bitwise-Hermitian matrix on the
// whole GPU.  State arrays from rows_init_kernel.  Returns QCH_ERR_UNSUPPORTED
// (caller falls back to the single-CTA driver) when a cooperative launch of
// one CTA per SM is not possible.
int npad_run_coop(double2* h, int n, double threshold, long long max_iter, int ek, const double* q, const int* c,
                  const double2* v, int* pivots, long long pivot_cap, long long* applied, int* status,
                  cudaStream_t st, double2* u) {
  int dev = 0, coop = 0;
  QCH_CUDA(cudaGetDevice(&dev));
  QCH_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  if (!coop) return QCH_ERR_UNSUPPORTED;
  // CTAs: the per-rotation time is mostly fixed latency (row reads, block
  // reductions, the record exchange), and every extra CTA adds a record to the
  // exchange.  Best measured: one 16-CTA cluster (records through DSMEM,
  // barrier.cluster) — dim 1024 5.6 us/rot, dim 4096 6.6 us/rot (32 CTAs
  // with global records: 7.9; 148: 11.2).  Without cluster support: n/128.
  int G = std::min(kClusterMax, std::max(1, n / 64));
  if (const char* ce = getenv("QCH_NPAD_COOP_CLUSTER"); ce != nullptr && atoi(ce) == 0)
    G = std::max(16, std::min(sm_count(), n / 128));
  if (const char* e = getenv("QCH_NPAD_COOP_CTAS")) G = std::max(1, std::min(sm_count(), atoi(e)));
  const int rows_per = (n + G - 1) / G;
  G = (n + rows_per - 1) / rows_per;
  const size_t smem = npad_coop_smem(n, rows_per);
  if (smem > (size_t)max_smem_optin()) return QCH_ERR_UNSUPPORTED;
  // one cluster of G <= 16 CTAs when the device can place it (QCH_NPAD_COOP_CLUSTER=0 disables)
  const char* ce = getenv("QCH_NPAD_COOP_CLUSTER");
  bool cl = (ce == nullptr || atoi(ce) != 0) && G <= kClusterMax;
  const bool stats_on = getenv("QCH_NPAD_STATS") != nullptr;
  auto pick = [&](bool cluster) {
    if (stats_on)
      return ek ? (cluster ? npad_coop_kernel<true, true, true> : npad_coop_kernel<true, false, true>)
                : (cluster ? npad_coop_kernel<false, true, true> : npad_coop_kernel<false, false, true>);
    return ek ? (cluster ? npad_coop_kernel<true, true, false> : npad_coop_kernel<true, false, false>)
              : (cluster ? npad_coop_kernel<false, true, false> : npad_coop_kernel<false, false, false>);
  };
  auto kern = pick(cl);
  QCH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (cl) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
      cudaGetLastError();
      cl = false;
    } else {
      cudaLaunchConfig_t qc = {};
      qc.gridDim = dim3(G);
      qc.blockDim = dim3(kCoopThreads);
      qc.dynamicSmemBytes = smem;
      cudaLaunchAttribute qa;
      qa.id = cudaLaunchAttributeClusterDimension;
      qa.val.clusterDim.x = G;
      qa.val.clusterDim.y = 1;
      qa.val.clusterDim.z = 1;
      qc.attrs = &qa;
      qc.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, (const void*)kern, &qc) != cudaSuccess || ncl < 1) {
        cudaGetLastError();
        cl = false;
      }
    }
    if (!cl) {
      kern = pick(false);
      QCH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
  }
  if (!cl) {
    int per_sm = 0;
    QCH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kCoopThreads, smem));
    if (per_sm < 1) return QCH_ERR_UNSUPPORTED;
  }

  void* ws = nullptr;
  ensure_pool();
  const size_t bytes = sizeof(CoopRec) * 2 * G + 256;
  QCH_CUDA(cudaMallocAsync(&ws, bytes, st));
  CoopArgs a;
  a.h = h;
  a.u = u;
  a.n = n;
  a.rows_per = rows_per;
  a.ek = ek;
  a.threshold = threshold;
  a.max_iter = max_iter;
  a.st_q = q;
  a.st_c = c;
  a.st_v = v;
  a.rec = (CoopRec*)ws;
  a.out_applied = (long long*)((char*)ws + sizeof(CoopRec) * 2 * G);
  a.out_status = (int*)(a.out_applied + 1);
  a.pivots = pivots;
  a.pivot_cap = pivot_cap;
  a.stats = nullptr;
  static const int mbx_env = getenv("QCH_NPAD_COOP_MBX") ? atoi(getenv("QCH_NPAD_COOP_MBX")) : 1;
  a.mbx = mbx_env;
  static const int pf_env = getenv("QCH_NPAD_COOP_PF") ? atoi(getenv("QCH_NPAD_COOP_PF")) : 1;
  a.pf_rescan = pf_env;
  static long long* d_cstats = nullptr;
  if (getenv("QCH_NPAD_STATS")) {
    if (d_cstats == nullptr) QCH_CUDA(cudaMalloc(&d_cstats, 8 * kMaxCoopCtas * sizeof(long long)));
    a.stats = d_cstats;
  }
  QCH_CUDA(cudaMemsetAsync(ws, 0xff, sizeof(CoopRec) * 2 * G, st));  // epochs = -1
  void* pr = prof_begin("npad_run_kernel", st);
  cudaError_t e;
  if (cl) {
    cudaLaunchConfig_t qc = {};
    qc.gridDim = dim3(G);
    qc.blockDim = dim3(kCoopThreads);
    qc.dynamicSmemBytes = smem;
    qc.stream = st;
    cudaLaunchAttribute qa;
    qa.id = cudaLaunchAttributeClusterDimension;
    qa.val.clusterDim.x = G;
    qa.val.clusterDim.y = 1;
    qa.val.clusterDim.z = 1;
    qc.attrs = &qa;
    qc.numAttrs = 1;
    e = cudaLaunchKernelEx(&qc, kern, a);
  } else {
    void* args[] = {&a};
    e = cudaLaunchCooperativeKernel((const void*)kern, dim3(G), dim3(kCoopThreads), args, smem, st);
  }
  prof_end(pr, st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    cudaFreeAsync(ws, st);
    return QCH_ERR_UNSUPPORTED;
  }
  note_launch(1);
  long long ap = 0;
  int stt = 0;
  QCH_CUDA(cudaMemcpyAsync(&ap, a.out_applied, sizeof ap, cudaMemcpyDeviceToHost, st));
  QCH_CUDA(cudaMemcpyAsync(&stt, a.out_status, sizeof stt, cudaMemcpyDeviceToHost, st));
  QCH_CUDA(cudaFreeAsync(ws, st));
  QCH_CUDA(cudaStreamSynchronize(st));
  *applied = ap;
  *status = stt;
  if (a.stats != nullptr && ap > 0) {
    std::vector<long long> hs(8 * (size_t)G);
    QCH_CUDA(cudaMemcpy(hs.data(), a.stats, hs.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    // CTA 0, then the max over CTAs of each phase (the slowest CTA sets the barrier)
    for (int row = 0; row < 2; ++row) {
      double v[8];
      for (int k = 0; k < 8; ++k) {
        v[k] = (double)hs[k] / ap;
        if (row == 1)
          for (int q = 1; q < G; ++q) v[k] = std::max(v[k], (double)hs[8 * q + k] / ap);
      }
      fprintf(stderr,
              "[qch npad coop] G=%d cluster=%d %s: cycles/rotation wait %.0f combine %.0f scalars %.0f rotate %.0f "
              "rescans %.0f (%.2f rows) own-best %.0f publish %.0f\n",
              G, cl ? 1 : 0, row == 0 ? "CTA 0" : "max  ", v[0], v[1], v[2], v[3], v[4], v[6], v[7], v[5]);
    }
  }
  return QCH_OK;
}

}  // namespace qch
