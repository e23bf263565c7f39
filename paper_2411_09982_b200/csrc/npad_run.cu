// npad_run.cu — the greedy NPAD driver (npad_run, npad.py:320-354) as ONE
// persistent thread block per matrix.  Two variants:
//
//  rows kernel   full-diagonal mode (and any subspace / non-bitwise-Hermitian
//                input): per-row maxima of the relevant strict lower triangle
//                in shared memory, maintained incrementally.  A rotation (i,j)
//                changes rows/columns i, j only: every other row folds in its
//                two new entries; rows whose stored argmax column was i or j
//                are rescanned cooperatively; rows i, j are reduced from the
//                freshly rotated values still in registers.  3 barriers per
//                rotation.
//
//  T-rows kernel subspace mode with a small target T (the parameter sweep):
//                the relevant couplings are exactly the entries H[t, x],
//                t in T, x not in T (one endpoint inside, npad.py:307-310), so
//                only |T| running maxima are kept ("T-rows").  Each rotation
//                (t, u) rescans T-row t from registers, folds column u into the
//                other T-rows, and rescans only T-rows whose argmax was u.
//                Selection over |T| candidates is done redundantly by every
//                warp: 2 barriers per rotation.
//
// Both use the certified |z|^2 keys of npad_select.cuh, so the pivot order is
// the reference's, and the same rotation arithmetic (qch_math.cuh) as the
// reference's _conjugate_dense.  Bitwise-Hermitian matrices (checked by
// qch_hermitian_exact_c128) are updated by reading rows only and writing the
// columns as conjugates: 96*N bytes per rotation.
#include <cstdlib>
#include <cstring>

#include "npad_run.h"
#include "npad_select.cuh"
#include "qch_internal.h"

namespace qch {

struct RotSc {
  double c;
  cplx s;
  Block2 blk;
};

constexpr int kList = 30;

__device__ __forceinline__ bool below_threshold(const Cand& p, double thr, bool ek) {
  // mag < threshold with mag the exact numpy |z| (npad.py:348)
  if (ek) return p.q < thr;
  const double t2 = thr * thr;
  if (p.q > t2 * (1.0 + kRel)) return false;
  if (p.q < t2 * (1.0 - kRel)) return true;
  return np_cabs_ool(p.v.x, p.v.y) < thr;
}

template <typename P>
__device__ __forceinline__ P* carve(unsigned char*& sp, size_t count) {
  P* p = (P*)sp;
  sp += (sizeof(P) * count + 15) & ~size_t(15);
  return p;
}

// ============================================================================
// rows kernel
template <int CPT, bool HERM, bool SMEMH>
__global__ void __launch_bounds__(512) npad_rows_kernel(NpadJob2* __restrict__ jobs, NpadCommon2 cm) {
  NpadJob2* job = jobs + blockIdx.x;
  const int n = cm.n;
  const int T = blockDim.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = T >> 5;
  const bool sub = cm.inT != nullptr;
  const bool ek = cm.ek != 0;
  double2* __restrict__ ug = job->u;
  const bool track = ug != nullptr;

  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* sp = smem;
  double2* s_v = carve<double2>(sp, n);
  double* s_q = carve<double>(sp, n);
  double* s_dg = carve<double>(sp, HERM ? n : 0);
  double2* s_dgc = carve<double2>(sp, HERM ? 0 : n);
  int* s_col = carve<int>(sp, n);
  int* s_slot = carve<int>(sp, n);
  int* s_list = carve<int>(sp, n);
  unsigned char* s_inT = carve<unsigned char>(sp, n);
  Cand* s_part = carve<Cand>(sp, (size_t)(kList + 2) * nw);
  Cand* s_w = carve<Cand>(sp, 32);
  cplx* s_lv = carve<cplx>(sp, 2 * kList);
  RotSc* s_sc = carve<RotSc>(sp, 1);
  int* s_cnt = carve<int>(sp, 4);

  double2* h;
  if (SMEMH) {
    double2* s_h = carve<double2>(sp, (size_t)n * n);
    const double2* hg = job->h;
    for (int k = tid; k < n * n; k += T) s_h[k] = hg[k];
    h = s_h;
  } else {
    h = job->h;
  }
  __syncthreads();
  for (int x = tid; x < n; x += T) {
    s_q[x] = job->st_q[x];
    s_col[x] = job->st_c[x];
    s_v[x] = job->st_v[x];
    s_slot[x] = -1;
    s_inT[x] = sub ? cm.inT[x] : 0;
    if (HERM)
      s_dg[x] = h[(size_t)x * n + x].x;
    else
      s_dgc[x] = h[(size_t)x * n + x];
  }
  if (tid == 0) s_cnt[0] = 0;
  __syncthreads();

  long long applied = job->applied;
  const double thr = job->threshold;
  int status = 0;
  auto rel = [&](int r, int c) { return !sub || (s_inT[r] != s_inT[c]); };

  while (true) {
    // ---- Phase 1: finalize partial rows, local best, warp winner
    Cand best = cand_none();
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const int x = tid + k * T;
      if (x < n) {
        const int sl = s_slot[x];
        if (sl >= 0) {
          Cand b = cand_none();
          for (int w = 0; w < nw; ++w) cand_take(b, s_part[sl * nw + w]);
          s_q[x] = b.q;
          s_col[x] = (b.q > 0.0) ? (int)(b.cr >> 16) : -1;
          s_v[x] = b.v;
          s_slot[x] = -1;
          if (b.q > 0.0) cand_take(best, b);
        } else if (s_q[x] > 0.0) {
          Cand c;
          c.q = s_q[x];
          c.m = -1.0;
          c.cr = ((unsigned)s_col[x] << 16) | (unsigned)x;
          c.v = s_v[x];
          cand_take(best, c);
        }
      }
    }
    {
      const int wl = warp_argmax(best);
      if (wl < 0) {
        if (lane == 0) s_w[warp] = cand_none();
      } else if (lane == wl) {
        s_w[warp] = best;
      }
    }
    __syncthreads();  // ---------------------------------------------- A

    // ---- Phase 2: global pick (every warp, redundantly), stop tests
    Cand pc = (lane < nw) ? s_w[lane] : cand_none();
    const int pl = warp_argmax(pc);
    const Cand piv = (pl >= 0) ? s_w[pl] : cand_none();
    if (applied >= cm.stop_at) {
      status = 2;
      break;
    }
    if (!(piv.q > 0.0) || below_threshold(piv, thr, ek)) {
      status = 0;
      break;
    }
    if (applied >= cm.max_iter) {
      status = 1;
      break;
    }
    const int i = (int)(piv.cr >> 16), j = (int)(piv.cr & 0xffffu);
    if (tid == 0) {
      const cplx v = d2c(piv.v);
      cplx hii, hjj, hij;
      if (HERM) {
        hii = mkc(s_dg[i], 0.0);
        hjj = mkc(s_dg[j], 0.0);
        hij = cconj(v);
      } else {
        hii = d2c(s_dgc[i]);
        hjj = d2c(s_dgc[j]);
        hij = d2c(h[(size_t)i * n + j]);
      }
      double c;
      cplx s;
      givens_fast(v, hii.re, hjj.re, &c, &s);
      s_sc->c = c;
      s_sc->s = s;
      s_sc->blk = rotate_block(c, s, hii, hij, v, hjj);
      if (job->pivots != nullptr && applied < job->pivot_cap) {
        job->pivots[2 * applied] = i;
        job->pivots[2 * applied + 1] = j;
      }
      s_slot[i] = 0;
      s_slot[j] = 1;
    }
    // rows whose stored argmax column is i or j are rescanned
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const int x = tid + k * T;
      if (x < n && x != i && x != j && s_q[x] > 0.0) {
        const int c = s_col[x];
        if (c == i || c == j) {
          if (sub && !s_inT[x] && cm.n_target <= 32) {
            s_slot[x] = -3;  // short row: owner rescans its target columns
          } else {
            const int q = atomicAdd(&s_cnt[0], 1);
            s_list[q] = x;
            s_slot[x] = (q < kList) ? 2 + q : -2;
          }
        }
      }
    }
    cplx ri[CPT], rj[CPT], ci[CPT], cj[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const int x = tid + k * T;
      if (x < n) {
        ri[k] = d2c(h[(size_t)i * n + x]);
        rj[k] = d2c(h[(size_t)j * n + x]);
        if (!HERM) {
          ci[k] = d2c(h[(size_t)x * n + i]);
          cj[k] = d2c(h[(size_t)x * n + j]);
        }
      }
    }
    __syncthreads();  // ---------------------------------------------- B

    // ---- Phase 3: rotate, fold, partials
    const double c = s_sc->c;
    const cplx s = s_sc->s;
    const int nlist = s_cnt[0];
    Cand pi = cand_none(), pj = cand_none();
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const int x = tid + k * T;
      if (x >= n || x == i || x == j) continue;
      cplx ni, nj, cxi, cxj;
      rotate_rows(c, s, ri[k], rj[k], &ni, &nj);
      if (HERM) {
        cxi = cconj(ni);
        cxj = cconj(nj);
      } else {
        rotate_cols(c, s, ci[k], cj[k], &cxi, &cxj);
      }
      h[(size_t)i * n + x] = c2d(ni);
      h[(size_t)j * n + x] = c2d(nj);
      h[(size_t)x * n + i] = c2d(cxi);
      h[(size_t)x * n + j] = c2d(cxj);
      if (x < i && rel(i, x)) cand_take(pi, make_cand(c2d(ni), ((unsigned)x << 16) | (unsigned)i, ek));
      if (x < j && rel(j, x)) cand_take(pj, make_cand(c2d(nj), ((unsigned)x << 16) | (unsigned)j, ek));
      const int sl = s_slot[x];
      if (sl >= 2) {
        s_lv[2 * (sl - 2)] = cxi;
        s_lv[2 * (sl - 2) + 1] = cxj;
      } else if (sl == -3) {
        // short subspace row (x outside T): its relevant columns are T
        Cand b = cand_none();
        for (int q = 0; q < cm.n_target; ++q) {
          const int t = cm.tlist[q];
          if (t >= x) break;
          const double2 v = (t == i) ? c2d(cxi) : (t == j) ? c2d(cxj) : h[(size_t)x * n + t];
          cand_take(b, make_cand(v, ((unsigned)t << 16) | (unsigned)x, ek));
        }
        s_q[x] = b.q;
        s_col[x] = (b.q > 0.0) ? (int)(b.cr >> 16) : -1;
        s_v[x] = b.v;
        s_slot[x] = -1;
      } else if (sl == -1) {
        Cand b;
        b.q = s_q[x];
        b.m = -1.0;
        b.cr = ((unsigned)s_col[x] << 16) | (unsigned)x;
        b.v = s_v[x];
        bool ch = false;
        if (i < x && rel(x, i)) {
          Cand cnd = make_cand(c2d(cxi), ((unsigned)i << 16) | (unsigned)x, ek);
          if (cand_better(cnd, b)) {
            b = cnd;
            ch = true;
          }
        }
        if (j < x && rel(x, j)) {
          Cand cnd = make_cand(c2d(cxj), ((unsigned)j << 16) | (unsigned)x, ek);
          if (cand_better(cnd, b)) {
            b = cnd;
            ch = true;
          }
        }
        if (ch) {
          s_q[x] = b.q;
          s_col[x] = (int)(b.cr >> 16);
          s_v[x] = b.v;
        }
      }
    }
    if (tid == 0) {
      const Block2 b = s_sc->blk;
      h[(size_t)i * n + i] = c2d(b.ii);
      h[(size_t)i * n + j] = c2d(b.ij);
      h[(size_t)j * n + i] = c2d(b.ji);
      h[(size_t)j * n + j] = c2d(b.jj);
      if (HERM) {
        s_dg[i] = b.ii.re;
        s_dg[j] = b.jj.re;
      } else {
        s_dgc[i] = c2d(b.ii);
        s_dgc[j] = c2d(b.jj);
      }
      if (rel(j, i)) cand_take(pj, make_cand(c2d(b.ji), ((unsigned)i << 16) | (unsigned)j, ek));
    }
    if (track) {
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const int x = tid + k * T;
        if (x >= n) continue;
        cplx ui = d2c(ug[(size_t)i * n + x]), uj = d2c(ug[(size_t)j * n + x]);
        cplx ni, nj;
        rotate_rows(c, s, ui, uj, &ni, &nj);
        ug[(size_t)i * n + x] = c2d(ni);
        ug[(size_t)j * n + x] = c2d(nj);
      }
    }
    {
      int wl = warp_argmax(pi);
      if (wl < 0) {
        if (lane == 0) s_part[0 * nw + warp] = cand_none();
      } else if (lane == wl) {
        s_part[0 * nw + warp] = pi;
      }
      wl = warp_argmax(pj);
      if (wl < 0) {
        if (lane == 0) s_part[1 * nw + warp] = cand_none();
      } else if (lane == wl) {
        s_part[1 * nw + warp] = pj;
      }
    }
    const int nl = nlist < kList ? nlist : kList;
    for (int q = 0; q < nl; ++q) {
      const int r = s_list[q];
      Cand pr = cand_none();
      double2 vals[CPT];
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const int x = tid + k * T;
        vals[k] = (x < r && x != i && x != j) ? h[(size_t)r * n + x] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const int x = tid + k * T;
        if (x < r && x != i && x != j && rel(r, x))
          cand_take(pr, make_cand(vals[k], ((unsigned)x << 16) | (unsigned)r, ek));
      }
      if ((r % T) == tid) {
        if (i < r && rel(r, i)) cand_take(pr, make_cand(c2d(s_lv[2 * q]), ((unsigned)i << 16) | (unsigned)r, ek));
        if (j < r && rel(r, j))
          cand_take(pr, make_cand(c2d(s_lv[2 * q + 1]), ((unsigned)j << 16) | (unsigned)r, ek));
      }
      const int wl = warp_argmax(pr);
      if (wl < 0) {
        if (lane == 0) s_part[(2 + q) * nw + warp] = cand_none();
      } else if (lane == wl) {
        s_part[(2 + q) * nw + warp] = pr;
      }
    }
    ++applied;
    if (cm.stats && tid == 0) {
      job->stats[0] += nlist;
      job->stats[1] += nlist > kList ? 1 : 0;
    }
    __syncthreads();  // ---------------------------------------------- C
    if (nlist > kList) {
      // overflow rows: one warp per row straight from memory
      for (int q = kList + warp; q < nlist; q += nw) {
        const int r = s_list[q];
        Cand b = cand_none();
        for (int x = lane; x < r; x += 32)
          if (rel(r, x)) cand_take(b, make_cand(h[(size_t)r * n + x], ((unsigned)x << 16) | (unsigned)r, ek));
        const int wl = warp_argmax(b);
        if (lane == (wl < 0 ? 0 : wl)) {
          s_q[r] = (wl < 0) ? 0.0 : b.q;
          s_col[r] = (wl < 0) ? -1 : (int)(b.cr >> 16);
          s_v[r] = b.v;
          s_slot[r] = -1;
        }
      }
      __syncthreads();
    }
    if (tid == 0) s_cnt[0] = 0;
  }

  __syncthreads();
  for (int x = tid; x < n; x += T) {
    job->st_q[x] = s_q[x];
    job->st_c[x] = s_col[x];
    job->st_v[x] = s_v[x];
  }
  if (SMEMH) {
    double2* hg = job->h;
    for (int k = tid; k < n * n; k += T) hg[k] = h[k];
  }
  if (tid == 0) {
    job->applied = applied;
    job->status = status;
    if (cm.stats)
      printf("npad rows[n=%d cpt=%d T=%d]: applied=%lld list_rows=%lld overflow_rot=%lld\n", n, CPT, T, applied,
             job->stats[0], job->stats[1]);
  }
}

// ============================================================================
// T-rows kernel (subspace mode, bitwise-Hermitian matrices, |T| <= 32)
__device__ __forceinline__ Cand trow_cand(double2 htx, int t, int x, bool ek) {
  // lower-triangle entry of the pair {t, x}: H[max, min]; |.| equal both ways
  const bool tl = t > x;
  const double2 v = tl ? htx : make_double2(htx.x, -htx.y);
  const unsigned cr = tl ? (((unsigned)x << 16) | (unsigned)t) : (((unsigned)t << 16) | (unsigned)x);
  return make_cand(v, cr, ek);
}
__device__ __forceinline__ int partner_of(unsigned cr, int t) {
  const int c = (int)(cr >> 16), r = (int)(cr & 0xffffu);
  return c == t ? r : c;
}

template <int CPT>
__global__ void __launch_bounds__(512) npad_trows_kernel(NpadJob2* __restrict__ jobs, NpadCommon2 cm) {
  NpadJob2* job = jobs + blockIdx.x;
  const int n = cm.n, nT = cm.n_target;
  const int T = blockDim.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = T >> 5;
  const bool ek = cm.ek != 0;

  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* sp = smem;
  double* s_dg = carve<double>(sp, n);
  int* s_kof = carve<int>(sp, n);  // x -> index in T, -1 outside
  Cand* s_tc = carve<Cand>(sp, 32);
  Cand* s_part = carve<Cand>(sp, (size_t)32 * nw);
  RotSc* s_sc = carve<RotSc>(sp, 1);
  double2* __restrict__ h = job->h;

  for (int x = tid; x < n; x += T) {
    s_dg[x] = h[(size_t)x * n + x].x;
    s_kof[x] = -1;
  }
  __syncthreads();
  for (int k = tid; k < nT; k += T) {
    s_kof[cm.tlist[k]] = k;
    Cand c;
    c.q = job->st_q[k];
    c.m = -1.0;
    c.cr = (unsigned)job->st_c[k];
    c.v = job->st_v[k];
    s_tc[k] = c;
  }
  __syncthreads();

  long long applied = job->applied;
  const double thr = job->threshold;
  int status = 0;
  unsigned fin_mask = 0;  // T-rows with partial slots pending (uniform)

  long long tc0 = 0, tc1 = 0, tc2 = 0, tc3 = 0;
  while (true) {
    if (cm.stats && tid == 0) tc0 = clock64();
    // ---- Phase 1 (every warp redundantly): finalize pending T-rows, select
    Cand mine = cand_none();
    if (lane < nT) {
      if ((fin_mask >> lane) & 1u) {
        for (int w = 0; w < nw; ++w) cand_take(mine, s_part[lane * nw + w]);
      } else {
        mine = s_tc[lane];
      }
    }
    const Cand my_tc = mine;
    // commit finalized T-rows: no warp reads s_tc for a pending lane this phase
    if (warp == 0 && lane < nT && ((fin_mask >> lane) & 1u)) s_tc[lane] = my_tc;
    const int pl = warp_argmax(mine);
    Cand piv = cand_none();
    if (pl >= 0) {
      piv.q = __shfl_sync(kFull, mine.q, pl);
      piv.m = __shfl_sync(kFull, mine.m, pl);
      piv.cr = __shfl_sync(kFull, mine.cr, pl);
      piv.v.x = __shfl_sync(kFull, mine.v.x, pl);
      piv.v.y = __shfl_sync(kFull, mine.v.y, pl);
    }
    if (applied >= cm.stop_at) {
      status = 2;
      break;
    }
    if (!(piv.q > 0.0) || below_threshold(piv, thr, ek)) {
      status = 0;
      break;
    }
    if (applied >= cm.max_iter) {
      status = 1;
      break;
    }
    if (cm.stats && tid == 0) tc1 = clock64();
    const int i = (int)(piv.cr >> 16), j = (int)(piv.cr & 0xffffu);
    const int kt = s_kof[i] >= 0 ? s_kof[i] : s_kof[j];
    const int t = cm.tlist[kt];
    const int u = (t == i) ? j : i;
    // T-rows (other than kt) whose argmax partner is u need a full rescan
    const unsigned resc = __ballot_sync(kFull, lane < nT && lane != kt && (my_tc.q > 0.0) &&
                                                   partner_of(my_tc.cr, cm.tlist[lane]) == u);
    if (tid == 0) {
      const cplx v = d2c(piv.v);
      double c;
      cplx s;
      givens_fast(v, s_dg[i], s_dg[j], &c, &s);
      s_sc->c = c;
      s_sc->s = s;
      s_sc->blk = rotate_block(c, s, mkc(s_dg[i], 0.0), cconj(v), v, mkc(s_dg[j], 0.0));
      if (job->pivots != nullptr && applied < job->pivot_cap) {
        job->pivots[2 * applied] = i;
        job->pivots[2 * applied + 1] = j;
      }
    }
    cplx ri[CPT], rj[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const int x = tid + k * T;
      if (x < n) {
        ri[k] = d2c(h[(size_t)i * n + x]);
        rj[k] = d2c(h[(size_t)j * n + x]);
      }
    }
    __syncthreads();  // ---------------------------------------------- B
    if (cm.stats && tid == 0) tc2 = clock64();

    // ---- Phase 3
    const double c = s_sc->c;
    const cplx s = s_sc->s;
    Cand pt = cand_none();  // T-row kt partial
    const bool t_is_i = (t == i);
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const int x = tid + k * T;
      if (x >= n || x == i || x == j) continue;
      cplx ni, nj;
      rotate_rows(c, s, ri[k], rj[k], &ni, &nj);
      h[(size_t)i * n + x] = c2d(ni);
      h[(size_t)j * n + x] = c2d(nj);
      h[(size_t)x * n + i] = c2d(cconj(ni));
      h[(size_t)x * n + j] = c2d(cconj(nj));
      const int kx = s_kof[x];
      if (kx < 0) {
        cand_take(pt, trow_cand(c2d(t_is_i ? ni : nj), t, x, ek));
      } else {
        // x = t' in T: the new H[t', u] = conj(new H[u, t']); T-rows being
        // rescanned get it in the rescan loop below
        if (!((resc >> kx) & 1u)) {
          const cplx nu = t_is_i ? nj : ni;
          Cand cnd = trow_cand(c2d(cconj(nu)), x, u, ek);
          Cand cur = s_tc[kx];
          if (cand_better(cnd, cur)) s_tc[kx] = cnd;
        }
      }
    }
    if (tid == 0) {
      const Block2 b = s_sc->blk;
      h[(size_t)i * n + i] = c2d(b.ii);
      h[(size_t)i * n + j] = c2d(b.ij);
      h[(size_t)j * n + i] = c2d(b.ji);
      h[(size_t)j * n + j] = c2d(b.jj);
      s_dg[i] = b.ii.re;
      s_dg[j] = b.jj.re;
      cand_take(pt, make_cand(c2d(b.ji), ((unsigned)i << 16) | (unsigned)j, ek));
    }
    {
      const int wl = warp_argmax(pt);
      if (wl < 0) {
        if (lane == 0) s_part[kt * nw + warp] = cand_none();
      } else if (lane == wl) {
        s_part[kt * nw + warp] = pt;
      }
    }
    // full rescans of the T-rows whose argmax partner was u
    unsigned rm = resc;
    while (rm) {
      const int kr = __ffs(rm) - 1;
      rm &= rm - 1;
      const int tr = cm.tlist[kr];
      Cand pr = cand_none();
      double2 vals[CPT];
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const int x = tid + k * T;
        vals[k] = (x < n && x != i && x != j && s_kof[x] < 0) ? h[(size_t)tr * n + x] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const int x = tid + k * T;
        if (x < n && x != i && x != j && s_kof[x] < 0) cand_take(pr, trow_cand(vals[k], tr, x, ek));
      }
      // entry (tr, u): the owner of column tr computed row u's new value there
      if ((tr % T) == tid) {
        const int kk = (tr - tid) / T;
        cplx nu = mkc(0, 0);
#pragma unroll
        for (int k = 0; k < CPT; ++k)
          if (k == kk) {
            cplx ni, nj;
            rotate_rows(c, s, ri[k], rj[k], &ni, &nj);
            nu = t_is_i ? nj : ni;
          }
        cand_take(pr, trow_cand(c2d(cconj(nu)), tr, u, ek));
      }
      const int wl = warp_argmax(pr);
      if (wl < 0) {
        if (lane == 0) s_part[kr * nw + warp] = cand_none();
      } else if (lane == wl) {
        s_part[kr * nw + warp] = pr;
      }
    }
    fin_mask = resc | (1u << kt);
    if (cm.stats && tid == 0) {
      tc3 = clock64();
      job->stats[0] += __popc(resc);
      job->stats[1] += tc1 - tc0;
      job->stats[2] += tc2 - tc1;
      job->stats[3] += tc3 - tc2;
    }
    ++applied;
    __syncthreads();  // ---------------------------------------------- C
  }

  __syncthreads();
  if (tid < nT) {
    job->st_q[tid] = s_tc[tid].q;
    job->st_c[tid] = (int)s_tc[tid].cr;
    job->st_v[tid] = s_tc[tid].v;
  }
  if (tid == 0) {
    job->applied = applied;
    job->status = status;
    if (cm.stats && blockIdx.x < 4)
      printf("trows[blk %d n=%d T=%d]: applied=%lld rescans=%lld cyc/rot: select=%lld prefetch+B=%lld update=%lld\n",
             blockIdx.x, n, T, applied, job->stats[0], job->stats[1] / (applied ? applied : 1),
             job->stats[2] / (applied ? applied : 1), job->stats[3] / (applied ? applied : 1));
  }
}

// ============================================================================
// initial candidate state
// rows: one warp per (matrix, row)
__global__ void rows_init_kernel(const double2* __restrict__ h, int n, const unsigned char* __restrict__ inT,
                                 const int* __restrict__ tlist, int nT, int ek, double* __restrict__ q,
                                 int* __restrict__ col, double2* __restrict__ val) {
  const int64_t b = blockIdx.y;
  const double2* hm = h + b * (int64_t)n * n;
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= n) return;
  Cand best = cand_none();
  if (inT != nullptr && !inT[r]) {
    for (int k = lane; k < nT; k += 32) {
      const int c = tlist[k];
      if (c < r) cand_take(best, make_cand(hm[(int64_t)r * n + c], ((unsigned)c << 16) | (unsigned)r, ek));
    }
  } else {
    for (int c = lane; c < r; c += 32) {
      if (inT != nullptr && inT[c]) continue;
      cand_take(best, make_cand(hm[(int64_t)r * n + c], ((unsigned)c << 16) | (unsigned)r, ek));
    }
  }
  const int wl = warp_argmax(best);
  if (lane == (wl < 0 ? 0 : wl)) {
    q[b * n + r] = (wl < 0) ? 0.0 : best.q;
    col[b * n + r] = (wl < 0) ? -1 : (int)(best.cr >> 16);
    val[b * n + r] = best.v;
  }
}

// T-rows: one warp per (matrix, target index)
__global__ void trows_init_kernel(const double2* __restrict__ h, int n, const unsigned char* __restrict__ inT,
                                  const int* __restrict__ tlist, int nT, int ek, double* __restrict__ q,
                                  int* __restrict__ crs, double2* __restrict__ val) {
  const int64_t b = blockIdx.y;
  const double2* hm = h + b * (int64_t)n * n;
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= nT) return;
  const int t = tlist[k];
  Cand best = cand_none();
  for (int x = lane; x < n; x += 32) {
    if (inT[x]) continue;
    cand_take(best, trow_cand(hm[(int64_t)t * n + x], t, x, ek));
  }
  const int wl = warp_argmax(best);
  if (lane == (wl < 0 ? 0 : wl)) {
    q[b * nT + k] = (wl < 0) ? 0.0 : best.q;
    crs[b * nT + k] = (wl < 0) ? -1 : (int)best.cr;
    val[b * nT + k] = best.v;
  }
}

// ============================================================================
// host-side launch helpers
static size_t rows_smem(int n, int threads, bool herm, bool smemh) {
  auto al = [](size_t b) { return (b + 15) & ~size_t(15); };
  const int nw = threads / 32;
  size_t s = al(16 * (size_t)n) + al(8 * (size_t)n) + (herm ? al(8 * (size_t)n) : al(16 * (size_t)n)) +
             3 * al(4 * (size_t)n) + al(n) + al(sizeof(Cand) * (kList + 2) * nw) + al(sizeof(Cand) * 32) +
             al(sizeof(cplx) * 2 * kList) + al(sizeof(RotSc)) + al(16);
  if (smemh) s += al(16 * (size_t)n * n);
  return s;
}
static size_t trows_smem(int n, int threads) {
  auto al = [](size_t b) { return (b + 15) & ~size_t(15); };
  const int nw = threads / 32;
  return al(8 * (size_t)n) + al(4 * (size_t)n) + al(sizeof(Cand) * 32) + al(sizeof(Cand) * 32 * nw) +
         al(sizeof(RotSc));
}

static void shape_for(int n, int pref, int* cpt, int* threads) {
  int c = 1;
  while (c < 8 && (n + c - 1) / c > pref) c *= 2;
  int t = ((n + c - 1) / c + 31) / 32 * 32;
  *cpt = c;
  *threads = t < 32 ? 32 : t;
}

template <int CPT, bool HERM, bool SMEMH>
static int launch_rows_t(NpadJob2* jobs, int njobs, const NpadCommon2& cm, int threads, cudaStream_t st) {
  size_t smem = rows_smem(cm.n, threads, HERM, SMEMH);
  if (smem > (size_t)max_smem_optin())
    return fail(QCH_ERR_UNSUPPORTED, "npad: dimension " + std::to_string(cm.n) + " needs " + std::to_string(smem) +
                                         " B of shared memory for the single-block driver");
  auto k = npad_rows_kernel<CPT, HERM, SMEMH>;
  QCH_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  void* pr = prof_begin("npad_run_kernel", st);
  k<<<njobs, threads, smem, st>>>(jobs, cm);
  prof_end(pr, st);
  QCH_LAUNCH_CHECK("npad_rows_kernel");
  note_launch(1);
  return QCH_OK;
}

template <int CPT>
static int launch_trows_t(NpadJob2* jobs, int njobs, const NpadCommon2& cm, int threads, cudaStream_t st) {
  size_t smem = trows_smem(cm.n, threads);
  if (smem > (size_t)max_smem_optin()) return fail(QCH_ERR_UNSUPPORTED, "npad: T-rows driver shared memory");
  auto k = npad_trows_kernel<CPT>;
  QCH_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  void* pr = prof_begin("npad_run_kernel", st);
  k<<<njobs, threads, smem, st>>>(jobs, cm);
  prof_end(pr, st);
  QCH_LAUNCH_CHECK("npad_trows_kernel");
  note_launch(1);
  return QCH_OK;
}

bool npad_use_trows(const NpadCommon2& cm, bool herm) { return herm && cm.inT != nullptr && cm.n_target <= 32; }

int npad_state_init(const double2* h, int64_t batch, const NpadCommon2& cm, bool trows, double* q, int* c,
                    double2* v, cudaStream_t st) {
  if (trows) {
    if (cm.n_target == 0) return QCH_OK;
    dim3 grid((cm.n_target + 7) / 8, (unsigned)batch);
    trows_init_kernel<<<grid, 256, 0, st>>>(h, cm.n, cm.inT, cm.tlist, cm.n_target, cm.ek, q, c, v);
    QCH_LAUNCH_CHECK("trows_init_kernel");
  } else {
    dim3 grid((cm.n + 7) / 8, (unsigned)batch);
    rows_init_kernel<<<grid, 256, 0, st>>>(h, cm.n, cm.inT, cm.tlist, cm.n_target, cm.ek, q, c, v);
    QCH_LAUNCH_CHECK("rows_init_kernel");
  }
  note_launch(1);
  return QCH_OK;
}

// single chain: widest useful block; batch: pref_threads per block
int npad_launch2(NpadJob2* jobs, int njobs, const NpadCommon2& cm, bool herm, bool trows, int pref_threads,
                 bool allow_smem_h, cudaStream_t st) {
  int cpt, threads;
  shape_for(cm.n, pref_threads, &cpt, &threads);
  // many independent chains (the sweep): one warp per chain with lazy
  // columns (npad_warp.cu); QCH_NPAD_DRIVER=warp|cta|tsmem|block overrides
  // (cta: npad_cta.cu; tsmem: npad_tsmem.cu, T-rows in shared memory)
  if (trows) {
    const char* d = getenv("QCH_NPAD_DRIVER");
    const char* wenv = getenv("QCH_NPAD_WARP");  // legacy switch: 1 = many-chain driver for any batch
    const bool many = wenv ? atoi(wenv) != 0 : njobs > 1;
    if (d != nullptr && strcmp(d, "warp") == 0) return npad_launch_trows_warp(jobs, njobs, cm, st);
    if (d != nullptr && strcmp(d, "cta") == 0) return npad_launch_trows_cta(jobs, njobs, cm, st);
    if (d != nullptr && strcmp(d, "tsmem") == 0 && npad_tsmem_bytes(cm) > 0) return npad_launch_tsmem(jobs, njobs, cm, st);
    if ((d == nullptr || strcmp(d, "block") != 0) && many) return npad_launch_trows_warp(jobs, njobs, cm, st);
  }
  if (npad_full_warp_ok(cm, herm, trows)) return npad_launch_full_warp(jobs, njobs, cm, st);
  if (trows) {
    switch (cpt) {
      case 1: return launch_trows_t<1>(jobs, njobs, cm, threads, st);
      case 2: return launch_trows_t<2>(jobs, njobs, cm, threads, st);
      case 4: return launch_trows_t<4>(jobs, njobs, cm, threads, st);
      default: return launch_trows_t<8>(jobs, njobs, cm, threads, st);
    }
  }
  const bool smemh = allow_smem_h && cpt == 1 && rows_smem(cm.n, threads, herm, true) <= (size_t)max_smem_optin();
  if (smemh) {
    return herm ? launch_rows_t<1, true, true>(jobs, njobs, cm, threads, st)
                : launch_rows_t<1, false, true>(jobs, njobs, cm, threads, st);
  }
  if (herm) {
    switch (cpt) {
      case 1: return launch_rows_t<1, true, false>(jobs, njobs, cm, threads, st);
      case 2: return launch_rows_t<2, true, false>(jobs, njobs, cm, threads, st);
      case 4: return launch_rows_t<4, true, false>(jobs, njobs, cm, threads, st);
      default: return launch_rows_t<8, true, false>(jobs, njobs, cm, threads, st);
    }
  }
  switch (cpt) {
    case 1: return launch_rows_t<1, false, false>(jobs, njobs, cm, threads, st);
    case 2: return launch_rows_t<2, false, false>(jobs, njobs, cm, threads, st);
    case 4: return launch_rows_t<4, false, false>(jobs, njobs, cm, threads, st);
    default: return launch_rows_t<8, false, false>(jobs, njobs, cm, threads, st);
  }
}

}  // namespace qch
