// npad.cu — NPAD (iterative Givens / Jacobi block diagonalisation) on sm_100a.
//
// Reference: /root/reference/pkg/src/effham/npad.py (+ operators.py for the
// container).  The greedy loop (npad_run, npad.py:320-354) is a serial chain:
// select the largest relevant coupling, rotate its 2x2 subspace, repeat.  We
// run the WHOLE chain inside one persistent thread block per matrix:
//
//  * selection (npad.py:300-317) is incremental: per-row maxima of the strict
//    lower triangle (magnitude desc, column asc) live in shared memory; a
//    rotation (i, j) changes only rows/columns i and j, so every other row
//    folds in its two new entries, and only rows whose stored argmax column
//    was i or j are rescanned.  The global pick is a block argmax over rows
//    with the reference tie-break (mag desc, i asc, j asc).  Magnitudes use
//    numpy's |z| rounding, so the pivot sequence is bit-identical.
//  * the rotation (npad.py:131-145) reads rows i and j once (coalesced,
//    16 B per lane), writes both rows and — because the matrix is bitwise
//    Hermitian — the two columns as conjugates of the new rows: 96*N bytes.
//  * 3 block barriers per rotation; the rotation scalars are computed by one
//    thread from shared-memory copies of the diagonal and of the pivot value
//    while the other threads prefetch rows i and j.
//
// One block per matrix makes the batched parameter sweep (many independent
// chains) fill the GPU; small matrices (N <= 112) are staged into shared
// memory for the single-chain case.
#include <cooperative_groups.h>

#include "qch_internal.h"
#include "qch_math.cuh"

namespace qch {

// ----------------------------------------------------------------------------
// packed selection key: (mag, cr = c<<16 | r); better = larger mag, then
// smaller (c, r).  Valid for N < 65536.
struct PKey {
  double mag;
  unsigned cr;
};
__device__ __forceinline__ PKey pk_none() { return PKey{-1.0, 0xffffffffu}; }
__device__ __forceinline__ bool pk_better(const PKey& a, const PKey& b) {
  return a.mag > b.mag || (a.mag == b.mag && a.cr < b.cr);
}
__device__ __forceinline__ PKey warp_best(PKey k) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    PKey o;
    o.mag = __shfl_xor_sync(0xffffffffu, k.mag, off);
    o.cr = __shfl_xor_sync(0xffffffffu, k.cr, off);
    if (pk_better(o, k)) k = o;
  }
  return k;
}
// row-local candidate compare: (mag desc, col asc)
__device__ __forceinline__ bool rowcand_better(double m1, int c1, double m2, int c2) {
  return m1 > m2 || (m1 == m2 && c1 < c2);
}

__device__ __forceinline__ double2 ld2(const double2* p) { return *p; }
__device__ __forceinline__ double2 ldg2(const double2* p) { return __ldcg(p); }

// ----------------------------------------------------------------------------
// max_abs (operators.py:92-99)
__global__ void max_abs_kernel(const double2* __restrict__ h, int64_t n, unsigned long long* out) {
  double m = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    double2 v = h[k];
    double a = np_cabs(v.x, v.y);
    m = fmax(m, a);  // NaN-ignoring max; finiteness is checked elsewhere
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  __shared__ double sm[32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sm[w] = m;
  __syncthreads();
  if (w == 0) {
    m = lane < (int)(blockDim.x >> 5) ? sm[lane] : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    // non-negative doubles order like their bit patterns
    if (lane == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
  }
}

__global__ void hermitian_exact_kernel(const double2* __restrict__ h, int64_t n, int* flag) {
  // sets *flag = 1 when some H[x,y] != conj(H[y,x])
  int64_t total = n * n;
  int bad = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    int64_t x = k / n, y = k - x * n;
    if (y > x) continue;
    double2 a = h[x * n + y], b = h[y * n + x];
    if (!(a.x == b.x && a.y == -b.y)) bad = 1;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// ----------------------------------------------------------------------------
// givens_rotation_matrix for a batch of pairs
__global__ void givens_params_kernel(const double2* __restrict__ h, int64_t n, const int64_t* __restrict__ pairs,
                                     int64_t np_, double* __restrict__ out, int* __restrict__ status) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= np_) return;
  int64_t i = pairs[2 * k], j = pairs[2 * k + 1];
  double2 v = h[j * n + i];
  double* o = out + 8 * k;
  if (v.x == 0.0 && v.y == 0.0) {
    status[k] = QCH_ERR_ZERO_COUPLING;
    for (int q = 0; q < 8; ++q) o[q] = 0.0;
    return;
  }
  status[k] = QCH_OK;
  RotParams p = givens_params(d2c(v), h[i * n + i].x, h[j * n + j].x);
  o[0] = p.cos_half;
  o[1] = p.sin_half;
  o[2] = p.phase;
  o[3] = p.degenerate ? 1.0 : 0.0;
  o[4] = p.s.re;
  o[5] = p.s.im;
  o[6] = 0.0;
  o[7] = 0.0;
}

// ----------------------------------------------------------------------------
// Apply P index-disjoint rotations in one launch with the reference's
// sequential semantics (eliminate_couplings applies them in list order,
// npad.py:291-296).  grid = (column chunks, P).  Entry (x, y) with x in pair p
// and y in pair q != p receives row-op p and column-op q in the order of the
// pair indices; all other entries receive one op.  Each block writes only the
// rows of its own pair (+ mirrored/updated columns at rows outside S).
__global__ void apply_rotations_kernel(double2* __restrict__ h, int64_t n, const int64_t* __restrict__ pairs,
                                       const double* __restrict__ params, int64_t np_, const int* __restrict__ pair_of,
                                       int herm, double2* __restrict__ u) {
  const int p = blockIdx.y;
  const int64_t i = pairs[2 * p], j = pairs[2 * p + 1];
  const double c = params[8 * p];
  const cplx s = mkc(params[8 * p + 4], params[8 * p + 5]);
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    int q = pair_of[x];
    if (q < 0) {
      cplx ri = d2c(h[i * n + x]), rj = d2c(h[j * n + x]);
      cplx ni, nj;
      rotate_rows(c, s, ri, rj, &ni, &nj);
      cplx ci, cj;
      if (herm) {
        ci = cconj(ni);
        cj = cconj(nj);
      } else {
        rotate_cols(c, s, d2c(h[x * n + i]), d2c(h[x * n + j]), &ci, &cj);
      }
      h[i * n + x] = c2d(ni);
      h[j * n + x] = c2d(nj);
      h[x * n + i] = c2d(ci);
      h[x * n + j] = c2d(cj);
    } else if (q == p) {
      if (x != i) continue;
      Block2 b = rotate_block(c, s, d2c(h[i * n + i]), d2c(h[i * n + j]), d2c(h[j * n + i]), d2c(h[j * n + j]));
      h[i * n + i] = c2d(b.ii);
      h[i * n + j] = c2d(b.ij);
      h[j * n + i] = c2d(b.ji);
      h[j * n + j] = c2d(b.jj);
    } else {
      const int64_t iq = pairs[2 * q], jq = pairs[2 * q + 1];
      if (x != iq) continue;  // the thread on column i_q handles both columns of pair q
      const double cq = params[8 * q];
      const cplx sq = mkc(params[8 * q + 4], params[8 * q + 5]);
      cplx a_ii = d2c(h[i * n + iq]), a_ij = d2c(h[i * n + jq]);  // row i_p at cols i_q, j_q
      cplx a_ji = d2c(h[j * n + iq]), a_jj = d2c(h[j * n + jq]);  // row j_p
      if (p < q) {
        // row op p (this pair) first, then column op q
        cplx r_ii, r_ji, r_ij, r_jj;
        rotate_rows(c, s, a_ii, a_ji, &r_ii, &r_ji);  // column i_q
        rotate_rows(c, s, a_ij, a_jj, &r_ij, &r_jj);  // column j_q
        rotate_cols(cq, sq, r_ii, r_ij, &a_ii, &a_ij);  // row i_p
        rotate_cols(cq, sq, r_ji, r_jj, &a_ji, &a_jj);  // row j_p
      } else {
        cplx t_ii, t_ij, t_ji, t_jj;
        rotate_cols(cq, sq, a_ii, a_ij, &t_ii, &t_ij);
        rotate_cols(cq, sq, a_ji, a_jj, &t_ji, &t_jj);
        rotate_rows(c, s, t_ii, t_ji, &a_ii, &a_ji);
        rotate_rows(c, s, t_ij, t_jj, &a_ij, &a_jj);
      }
      h[i * n + iq] = c2d(a_ii);
      h[i * n + jq] = c2d(a_ij);
      h[j * n + iq] = c2d(a_ji);
      h[j * n + jq] = c2d(a_jj);
    }
  }
  if (u != nullptr) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
      cplx ui = d2c(u[i * n + x]), uj = d2c(u[j * n + x]);
      cplx ni, nj;
      rotate_rows(c, s, ui, uj, &ni, &nj);
      u[i * n + x] = c2d(ni);
      u[j * n + x] = c2d(nj);
    }
  }
}

// ----------------------------------------------------------------------------
// Initial per-row maxima of the relevant strict lower triangle: one warp/row.
__device__ __forceinline__ bool relevant(const unsigned char* inT, int r, int c) {
  return inT == nullptr || (inT[r] != inT[c]);
}

__global__ void rowmax_init_kernel(const double2* __restrict__ h, int n, const unsigned char* __restrict__ inT,
                                   const int* __restrict__ tlist, int n_target, double* __restrict__ rmag,
                                   int* __restrict__ rcol, double2* __restrict__ rval) {
  // blockIdx.y = matrix in batch; state arrays are (batch, n)
  const double2* hm = h + (int64_t)blockIdx.y * n * n;
  double* rm = rmag + (int64_t)blockIdx.y * n;
  int* rc = rcol + (int64_t)blockIdx.y * n;
  double2* rv = rval + (int64_t)blockIdx.y * n;
  int lane = threadIdx.x & 31;
  int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= n) return;
  double bm = -1.0;
  int bc = 0x7fffffff;
  double2 bv = make_double2(0.0, 0.0);
  if (inT != nullptr && !inT[r]) {
    // subspace mode, row outside the target: only target columns are relevant
    for (int q = lane; q < n_target; q += 32) {
      int c = tlist[q];
      if (c >= r) continue;
      double2 v = hm[(int64_t)r * n + c];
      double m = np_cabs(v.x, v.y);
      if (rowcand_better(m, c, bm, bc)) {
        bm = m;
        bc = c;
        bv = v;
      }
    }
  } else {
    for (int c = lane; c < r; c += 32) {
      if (inT != nullptr && inT[c]) continue;
      double2 v = hm[(int64_t)r * n + c];
      double m = np_cabs(v.x, v.y);
      if (rowcand_better(m, c, bm, bc)) {
        bm = m;
        bc = c;
        bv = v;
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    double om = __shfl_xor_sync(0xffffffffu, bm, off);
    int oc = __shfl_xor_sync(0xffffffffu, bc, off);
    double ovx = __shfl_xor_sync(0xffffffffu, bv.x, off);
    double ovy = __shfl_xor_sync(0xffffffffu, bv.y, off);
    if (rowcand_better(om, oc, bm, bc)) {
      bm = om;
      bc = oc;
      bv = make_double2(ovx, ovy);
    }
  }
  if (lane == 0) {
    rm[r] = bm;
    rc[r] = (bm < 0.0) ? -1 : bc;
    rv[r] = bv;
  }
}

__global__ void fill_mask_kernel(unsigned char* mask, int n, const int* tlist, int nt) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) mask[x] = 0;
}
__global__ void set_mask_kernel(unsigned char* mask, const int* tlist, int nt) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nt; q += gridDim.x * blockDim.x) mask[tlist[q]] = 1;
}

// ----------------------------------------------------------------------------
// The greedy driver.  One block per job.
struct NpadJob {
  double2* h;        // (N,N)
  double2* u;        // accumulated unitary or nullptr
  double* rmag;      // persisted row-max state (N)
  int* rcol;         // (N)
  double2* rval;     // (N)
  int* pivots;       // 2*pivot_cap or nullptr
  long long pivot_cap;
  double threshold;
  long long applied;  // in: already applied; out: total applied
  int status;         // out: 0 converged, 1 max_iter reached, 2 paused at stop_at
};

struct NpadCommon {
  int n;
  const unsigned char* inT;  // nullptr: full-diagonal mode
  const int* tlist;          // sorted target list (subspace mode)
  int n_target;
  int herm;                  // 1: matrix is bitwise Hermitian
  int stage_h;               // 1: stage H in shared memory
  long long max_iter;
  long long stop_at;
};

constexpr int kListCap = 30;  // long rescan rows per rotation handled in-phase

struct NpadScalars {
  double c;
  cplx s;
  Block2 blk;
  int i, j;
};

template <int CPT>
__global__ void __launch_bounds__(1024) npad_run_kernel(NpadJob* __restrict__ jobs, NpadCommon cm) {
  NpadJob* job = jobs + blockIdx.x;
  const int n = cm.n;
  const int T = blockDim.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = T >> 5;
  const bool sub = cm.inT != nullptr;
  const bool herm = cm.herm != 0;
  double2* __restrict__ ug = job->u;
  const bool track = ug != nullptr;

  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* sp = smem;
  auto carve = [&](size_t bytes) {
    unsigned char* p = sp;
    sp += (bytes + 15) & ~size_t(15);
    return p;
  };
  double2* s_rval = (double2*)carve(sizeof(double2) * n);
  double* s_rmag = (double*)carve(sizeof(double) * n);
  double* s_diag = (double*)carve(sizeof(double) * n);
  int* s_rcol = (int*)carve(sizeof(int) * n);
  int* s_slot = (int*)carve(sizeof(int) * n);
  int* s_list = (int*)carve(sizeof(int) * n);
  unsigned char* s_inT = (unsigned char*)carve(n);
  PKey* s_part = (PKey*)carve(sizeof(PKey) * (kListCap + 2) * nw);
  PKey* s_wkey = (PKey*)carve(sizeof(PKey) * 32);
  cplx* s_lv = (cplx*)carve(sizeof(cplx) * 2 * kListCap);
  NpadScalars* s_sc = (NpadScalars*)carve(sizeof(NpadScalars));
  int* s_cnt = (int*)carve(sizeof(int) * 4);
  double2* s_h = cm.stage_h ? (double2*)carve(sizeof(double2) * (size_t)n * n) : nullptr;

  double2* __restrict__ h = job->h;
  if (cm.stage_h) {
    for (int k = tid; k < n * n; k += T) s_h[k] = h[k];
    h = s_h;
  }
  for (int x = tid; x < n; x += T) {
    s_rmag[x] = job->rmag[x];
    s_rcol[x] = job->rcol[x];
    s_rval[x] = job->rval[x];
    s_slot[x] = -1;
    s_inT[x] = sub ? cm.inT[x] : 0;
    s_diag[x] = herm ? (cm.stage_h ? s_h[(size_t)x * n + x].x : h[(size_t)x * n + x].x) : 0.0;
  }
  if (tid == 0) s_cnt[0] = 0;
  __syncthreads();

  long long applied = job->applied;
  const double threshold = job->threshold;
  int status = 0;

  // rows owned by this thread: x = tid + k*T, k < CPT
  while (true) {
    // ---------------- Phase 1: finalize partial rows, local best, warp best
    PKey best = pk_none();
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      int x = tid + k * T;
      if (x < n) {
        int sl = s_slot[x];
        if (sl >= 0) {
          PKey b = pk_none();
          for (int w = 0; w < nw; ++w) {
            PKey o = s_part[sl * nw + w];
            if (pk_better(o, b)) b = o;
          }
          if (b.mag >= 0.0) {
            int c = (int)(b.cr >> 16);
            s_rmag[x] = b.mag;
            s_rcol[x] = c;
            s_rval[x] = h[(size_t)x * n + c];
          } else {
            s_rmag[x] = -1.0;
            s_rcol[x] = -1;
          }
          s_slot[x] = -1;
        }
        double m = s_rmag[x];
        if (m >= 0.0) {
          PKey kk{m, ((unsigned)s_rcol[x] << 16) | (unsigned)x};
          if (pk_better(kk, best)) best = kk;
        }
      }
    }
    best = warp_best(best);
    if (lane == 0) s_wkey[warp] = best;
    __syncthreads();  // ---- A

    // ---------------- Phase 2: global pick, stop tests, scalars, prefetch
    PKey piv = lane < nw ? s_wkey[lane] : pk_none();
    piv = warp_best(piv);
    if (applied >= cm.stop_at) {
      status = 2;
      break;
    }
    if (piv.mag <= 0.0 || piv.mag < threshold) {  // None or below threshold
      status = 0;
      break;
    }
    if (applied >= cm.max_iter) {
      status = 1;
      break;
    }
    const int i = (int)(piv.cr >> 16), j = (int)(piv.cr & 0xffffu);
    if (tid == 0) {
      cplx hji = d2c(s_rval[j]);
      cplx hij, hii, hjj;
      double dii, djj;
      if (herm) {
        dii = s_diag[i];
        djj = s_diag[j];
        hii = mkc(dii, 0.0);
        hjj = mkc(djj, 0.0);
        hij = cconj(hji);
      } else {
        hii = d2c(h[(size_t)i * n + i]);
        hjj = d2c(h[(size_t)j * n + j]);
        hij = d2c(h[(size_t)i * n + j]);
        dii = hii.re;
        djj = hjj.re;
      }
      RotParams rp = givens_params(hji, dii, djj);
      s_sc->c = rp.cos_half;
      s_sc->s = rp.s;
      s_sc->blk = rotate_block(rp.cos_half, rp.s, hii, hij, hji, hjj);
      if (job->pivots != nullptr && applied < job->pivot_cap) {
        job->pivots[2 * applied] = i;
        job->pivots[2 * applied + 1] = j;
      }
      s_slot[i] = 0;
      s_slot[j] = 1;
    }
    // rows whose stored argmax column is i or j need a rescan
    bool local_rescan[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      local_rescan[k] = false;
      int x = tid + k * T;
      if (x < n && x != i && x != j) {
        int rc = s_rcol[x];
        if (rc == i || rc == j) {
          bool shortrow = sub && !s_inT[x] && cm.n_target <= 32;
          if (shortrow) {
            local_rescan[k] = true;
          } else {
            int q = atomicAdd(&s_cnt[0], 1);
            s_list[q] = x;
            s_slot[x] = (q < kListCap) ? 2 + q : -2;
          }
        }
      }
    }
    cplx ri[CPT], rj[CPT], ci[CPT], cj[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      int x = tid + k * T;
      if (x < n) {
        ri[k] = d2c(h[(size_t)i * n + x]);
        rj[k] = d2c(h[(size_t)j * n + x]);
        if (!herm) {
          ci[k] = d2c(h[(size_t)x * n + i]);
          cj[k] = d2c(h[(size_t)x * n + j]);
        }
      }
    }
    __syncthreads();  // ---- B

    // ---------------- Phase 3: rotate, fold, partials
    const double c = s_sc->c;
    const cplx s = s_sc->s;
    const int nlist = s_cnt[0];
    const bool in_i = s_inT[i], in_j = s_inT[j];
    PKey pi = pk_none(), pj = pk_none();
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      int x = tid + k * T;
      if (x >= n || x == i || x == j) continue;
      cplx ni, nj, cxi, cxj;
      rotate_rows(c, s, ri[k], rj[k], &ni, &nj);
      if (herm) {
        cxi = cconj(ni);
        cxj = cconj(nj);
      } else {
        rotate_cols(c, s, ci[k], cj[k], &cxi, &cxj);
      }
      h[(size_t)i * n + x] = c2d(ni);
      h[(size_t)j * n + x] = c2d(nj);
      h[(size_t)x * n + i] = c2d(cxi);
      h[(size_t)x * n + j] = c2d(cxj);
      const bool in_x = s_inT[x];
      // rows i / j partials: entries (i,x), x<i and (j,x), x<j
      if (x < i && (!sub || in_i != in_x)) {
        PKey kk{np_cabs(ni), ((unsigned)x << 16) | (unsigned)i};
        if (pk_better(kk, pi)) pi = kk;
      }
      if (x < j && (!sub || in_j != in_x)) {
        PKey kk{np_cabs(nj), ((unsigned)x << 16) | (unsigned)j};
        if (pk_better(kk, pj)) pj = kk;
      }
      // row x: entries (x,i) if i<x, (x,j) if j<x
      bool rel_i = (i < x) && (!sub || in_i != in_x);
      bool rel_j = (j < x) && (!sub || in_j != in_x);
      int sl = s_slot[x];
      if (sl >= 2) {
        s_lv[2 * (sl - 2)] = cxi;  // new (x,i), (x,j) for the list-row partial
        s_lv[2 * (sl - 2) + 1] = cxj;
      } else if (sl == -2) {
        // overflow row: rescanned after barrier C from memory
      } else if (local_rescan[k]) {
        // short subspace row (x not in target): scan its target columns
        double bm = -1.0;
        int bc = -1;
        cplx bv = mkc(0, 0);
        for (int q = 0; q < cm.n_target; ++q) {
          int t = cm.tlist[q];
          if (t >= x) break;
          cplx v = (t == i) ? cxi : (t == j) ? cxj : d2c(h[(size_t)x * n + t]);
          double m = np_cabs(v);
          if (rowcand_better(m, t, bm, bc)) {
            bm = m;
            bc = t;
            bv = v;
          }
        }
        s_rmag[x] = bm;
        s_rcol[x] = bc;
        s_rval[x] = c2d(bv);
      } else {
        double bm = s_rmag[x];
        int bc = s_rcol[x];
        bool ch = false;
        cplx bv;
        if (rel_i) {
          double m = np_cabs(cxi);
          if (rowcand_better(m, i, bm, bc)) {
            bm = m;
            bc = i;
            bv = cxi;
            ch = true;
          }
        }
        if (rel_j) {
          double m = np_cabs(cxj);
          if (rowcand_better(m, j, bm, bc)) {
            bm = m;
            bc = j;
            bv = cxj;
            ch = true;
          }
        }
        if (ch) {
          s_rmag[x] = bm;
          s_rcol[x] = bc;
          s_rval[x] = c2d(bv);
        }
      }
    }
    if (tid == 0) {
      const Block2 b = s_sc->blk;
      h[(size_t)i * n + i] = c2d(b.ii);
      h[(size_t)i * n + j] = c2d(b.ij);
      h[(size_t)j * n + i] = c2d(b.ji);
      h[(size_t)j * n + j] = c2d(b.jj);
      s_diag[i] = b.ii.re;
      s_diag[j] = b.jj.re;
      if (!sub || in_i != in_j) {
        PKey kk{np_cabs(b.ji), ((unsigned)i << 16) | (unsigned)j};
        if (pk_better(kk, pj)) pj = kk;
      }
    }
    if (track) {
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        int x = tid + k * T;
        if (x >= n) continue;
        cplx ui = d2c(ug[(size_t)i * n + x]), uj = d2c(ug[(size_t)j * n + x]);
        cplx ni, nj;
        rotate_rows(c, s, ui, uj, &ni, &nj);
        ug[(size_t)i * n + x] = c2d(ni);
        ug[(size_t)j * n + x] = c2d(nj);
      }
    }
    pi = warp_best(pi);
    pj = warp_best(pj);
    if (lane == 0) {
      s_part[0 * nw + warp] = pi;
      s_part[1 * nw + warp] = pj;
    }
    // list rows: partial scans over owned columns
    const int nl = nlist < kListCap ? nlist : kListCap;
    for (int q = 0; q < nl; ++q) {
      const int r = s_list[q];
      const bool in_r = s_inT[r];
      PKey pr = pk_none();
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        int x = tid + k * T;
        if (x >= r || x == i || x == j) continue;
        if (sub && in_r == (bool)s_inT[x]) continue;
        double2 v = h[(size_t)r * n + x];
        PKey kk{np_cabs(v.x, v.y), ((unsigned)x << 16) | (unsigned)r};
        if (pk_better(kk, pr)) pr = kk;
      }
      if ((r % T) == tid) {
        // owner adds the entries it rotated: (r,i), (r,j)
        if (i < r && (!sub || in_r != in_i)) {
          PKey kk{np_cabs(s_lv[2 * q]), ((unsigned)i << 16) | (unsigned)r};
          if (pk_better(kk, pr)) pr = kk;
        }
        if (j < r && (!sub || in_r != in_j)) {
          PKey kk{np_cabs(s_lv[2 * q + 1]), ((unsigned)j << 16) | (unsigned)r};
          if (pk_better(kk, pr)) pr = kk;
        }
      }
      pr = warp_best(pr);
      if (lane == 0) s_part[(2 + q) * nw + warp] = pr;
    }
    ++applied;
    __syncthreads();  // ---- C
    if (nlist > kListCap) {
      // overflow: one warp per remaining row, straight from memory
      for (int q = kListCap + warp; q < nlist; q += nw) {
        const int r = s_list[q];
        const bool in_r = s_inT[r];
        double bm = -1.0;
        int bc = 0x7fffffff;
        for (int x = lane; x < r; x += 32) {
          if (sub && in_r == (bool)s_inT[x]) continue;
          double2 v = h[(size_t)r * n + x];
          double m = np_cabs(v.x, v.y);
          if (rowcand_better(m, x, bm, bc)) {
            bm = m;
            bc = x;
          }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          double om = __shfl_xor_sync(0xffffffffu, bm, off);
          int oc = __shfl_xor_sync(0xffffffffu, bc, off);
          if (rowcand_better(om, oc, bm, bc)) {
            bm = om;
            bc = oc;
          }
        }
        if (lane == 0) {
          s_rmag[r] = bm;
          s_rcol[r] = bm >= 0.0 ? bc : -1;
          if (bm >= 0.0) s_rval[r] = h[(size_t)r * n + bc];
          s_slot[r] = -1;
        }
      }
      __syncthreads();
    }
    if (tid == 0) s_cnt[0] = 0;
    // s_cnt reset is ordered before the next phase-2 atomics by barrier A
  }

  // ---------------- write back
  __syncthreads();
  for (int x = tid; x < n; x += T) {
    job->rmag[x] = s_rmag[x];
    job->rcol[x] = s_rcol[x];
    job->rval[x] = s_rval[x];
  }
  if (cm.stage_h) {
    double2* hg = job->h;
    for (int k = tid; k < n * n; k += T) hg[k] = s_h[k];
  }
  if (tid == 0) {
    job->applied = applied;
    job->status = status;
  }
}

// ----------------------------------------------------------------------------
// transmon (x) resonator builder
__global__ void build_tr_kernel(double2* __restrict__ h, int64_t nq, int64_t nr, const double* __restrict__ prm) {
  const int64_t n = nq * nr;
  const int64_t b = blockIdx.y;
  const double wq = prm[4 * b], al = prm[4 * b + 1], wr = prm[4 * b + 2], g = prm[4 * b + 3];
  double2* hb = h + b * n * n;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n * n; k += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = k / n, c = k - r * n;
    int64_t q1 = r / nr, k1 = r - q1 * nr, q2 = c / nr, k2 = c - q2 * nr;
    double v = 0.0;
    if (r == c) {
      // host builder (models.transmon_resonator_hamiltonian): n = b^dag b has
      // diagonal sqrt(q)^2 (not exactly q), a^dag a likewise; same op order.
      double sq = sqrt((double)q1), sk = sqrt((double)k1);
      double nn = QMUL(sq, sq), kk = QMUL(sk, sk);
      double hq = QADD(QMUL(wq, nn), QMUL(QMUL(0.5, al), QMUL(nn, QSUB(nn, 1.0))));
      v = QADD(hq, QMUL(wr, kk));
    } else {
      int64_t dq = q1 - q2, dk = k1 - k2;
      if ((dq == 1 || dq == -1) && (dk == 1 || dk == -1)) {
        double bq = sqrt((double)(q1 > q2 ? q1 : q2));
        double ak = sqrt((double)(k1 > k2 ? k1 : k2));
        v = QMUL(g, QMUL(bq, ak));
      }
    }
    hb[k] = make_double2(v, 0.0);
  }
}

}  // namespace qch

// ============================================================================
// host side
namespace qch {

static size_t npad_smem_bytes(int n, int threads, bool stage) {
  auto al = [](size_t b) { return (b + 15) & ~size_t(15); };
  int nw = threads / 32;
  size_t s = al(16 * (size_t)n) + al(8 * (size_t)n) + al(8 * (size_t)n) + 3 * al(4 * (size_t)n) + al(n) +
             al(sizeof(PKey) * (kListCap + 2) * nw) + al(sizeof(PKey) * 32) + al(sizeof(cplx) * 2 * kListCap) +
             al(sizeof(NpadScalars)) + al(16);
  if (stage) s += al(16 * (size_t)n * n);
  return s;
}

using npad_kernel_t = void (*)(NpadJob*, NpadCommon);

static npad_kernel_t npad_kernel_for(int cpt) {
  switch (cpt) {
    case 1: return npad_run_kernel<1>;
    case 2: return npad_run_kernel<2>;
    case 4: return npad_run_kernel<4>;
    case 8: return npad_run_kernel<8>;
    default: return nullptr;
  }
}

// pick (columns per thread, threads): single chains use the widest block
// (latency); batches use `pref_threads` so several chains share an SM.
static void npad_shape(int n, int pref_threads, int* cpt, int* threads) {
  int c = 1;
  while (c < 8 && (n + c - 1) / c > pref_threads) c *= 2;
  int t = (n + c - 1) / c;
  t = ((t + 31) / 32) * 32;
  if (t < 32) t = 32;
  *cpt = c;
  *threads = t;
}

struct Workspace {
  cudaStream_t st;
  void* p = nullptr;
  explicit Workspace(cudaStream_t s) : st(s) {}
  cudaError_t alloc(size_t bytes) { return cudaMallocAsync(&p, bytes, st); }
  ~Workspace() {
    if (p) cudaFreeAsync(p, st);
  }
};

int npad_launch(NpadJob* d_jobs, int njobs, NpadCommon cm, int pref_threads, cudaStream_t st) {
  int cpt, threads;
  npad_shape(cm.n, pref_threads, &cpt, &threads);
  npad_kernel_t k = npad_kernel_for(cpt);
  if (!k) return fail(QCH_ERR_UNSUPPORTED, "npad: dimension too large for the single-block driver");
  size_t smem = npad_smem_bytes(cm.n, threads, cm.stage_h != 0);
  if (smem > (size_t)max_smem_optin())
    return fail(QCH_ERR_UNSUPPORTED, "npad: dimension " + std::to_string(cm.n) + " needs " + std::to_string(smem) +
                                         " B of shared memory (max " + std::to_string(max_smem_optin()) + ")");
  QCH_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  void* pr = prof_begin("npad_run_kernel", st);
  k<<<njobs, threads, smem, st>>>(d_jobs, cm);
  prof_end(pr, st);
  QCH_LAUNCH_CHECK("npad_run_kernel");
  note_launch(1);
  return QCH_OK;
}

}  // namespace qch

using namespace qch;

extern "C" int qch_max_abs_c128(const void* d_h, int64_t n_elems, double* d_out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  QCH_CUDA(cudaMemsetAsync(d_out, 0, sizeof(double), st));
  if (n_elems <= 0) return QCH_OK;
  int blocks = (int)std::min<int64_t>((n_elems + 255) / 256, (int64_t)sm_count() * 8);
  max_abs_kernel<<<blocks, 256, 0, st>>>((const double2*)d_h, n_elems, (unsigned long long*)d_out);
  QCH_LAUNCH_CHECK("max_abs_kernel");
  note_launch(1);
  return QCH_OK;
}

extern "C" int qch_hermitian_exact_c128(const void* d_h, int64_t n, int* d_nonherm, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  QCH_CUDA(cudaMemsetAsync(d_nonherm, 0, sizeof(int), st));
  if (n <= 0) return QCH_OK;
  int blocks = (int)std::min<int64_t>((n * n + 255) / 256, (int64_t)sm_count() * 8);
  hermitian_exact_kernel<<<blocks, 256, 0, st>>>((const double2*)d_h, n, d_nonherm);
  QCH_LAUNCH_CHECK("hermitian_exact_kernel");
  note_launch(1);
  return QCH_OK;
}

extern "C" int qch_givens_params_c128(const void* d_h, int64_t n, const int64_t* d_pairs, int64_t n_pairs,
                                      double* d_params, int* d_status, void* stream) {
  if (n_pairs <= 0) return QCH_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int blocks = (int)((n_pairs + 127) / 128);
  givens_params_kernel<<<blocks, 128, 0, st>>>((const double2*)d_h, n, d_pairs, n_pairs, d_params, d_status);
  QCH_LAUNCH_CHECK("givens_params_kernel");
  note_launch(1);
  return QCH_OK;
}

__global__ void pair_of_kernel(int* pair_of, int64_t n, const int64_t* pairs, int64_t np_) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
    pair_of[x] = -1;
}
__global__ void pair_mark_kernel(int* pair_of, const int64_t* pairs, int64_t np_) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np_; p += (int64_t)gridDim.x * blockDim.x) {
    pair_of[pairs[2 * p]] = (int)p;
    pair_of[pairs[2 * p + 1]] = (int)p;
  }
}

extern "C" int qch_npad_apply_rotations_c128(void* d_h, int64_t n, const int64_t* d_pairs, const double* d_params,
                                             int64_t n_pairs, int herm_exact, void* d_u, void* stream) {
  if (n_pairs <= 0) return QCH_OK;
  if (n_pairs > 65535) return fail(QCH_ERR_UNSUPPORTED, "too many pairs in one launch");
  cudaStream_t st = (cudaStream_t)stream;
  Workspace ws(st);
  QCH_CUDA(ws.alloc(sizeof(int) * n));
  int* pair_of = (int*)ws.p;
  int b1 = (int)std::min<int64_t>((n + 255) / 256, 1024);
  pair_of_kernel<<<b1, 256, 0, st>>>(pair_of, n, d_pairs, n_pairs);
  pair_mark_kernel<<<(int)((n_pairs + 255) / 256), 256, 0, st>>>(pair_of, d_pairs, n_pairs);
  int chunks = (int)std::min<int64_t>((n + 255) / 256, std::max<int64_t>(1, (int64_t)sm_count() * 4 / n_pairs));
  dim3 grid(chunks, (unsigned)n_pairs);
  apply_rotations_kernel<<<grid, 256, 0, st>>>((double2*)d_h, n, d_pairs, d_params, n_pairs, pair_of, herm_exact,
                                               (double2*)d_u);
  QCH_LAUNCH_CHECK("apply_rotations_kernel");
  note_launch(3);
  return QCH_OK;
}

extern "C" int qch_build_transmon_resonator_c128(void* d_h, int64_t batch, int64_t n_q, int64_t n_r,
                                                 const double* d_params, void* stream) {
  if (batch <= 0) return QCH_OK;
  if (n_q < 1 || n_r < 1) return fail(QCH_ERR_VALUE, "need n_q, n_r >= 1");
  cudaStream_t st = (cudaStream_t)stream;
  int64_t n = n_q * n_r;
  int bx = (int)std::min<int64_t>((n * n + 255) / 256, std::max<int64_t>(1, (int64_t)sm_count() * 8 / batch + 1));
  dim3 grid(bx, (unsigned)batch);
  build_tr_kernel<<<grid, 256, 0, st>>>((double2*)d_h, n_q, n_r, d_params);
  QCH_LAUNCH_CHECK("build_tr_kernel");
  note_launch(1);
  return QCH_OK;
}

// shared setup of the npad drivers: mask, row-max state, jobs
static int npad_setup(const double2* d_h, int64_t batch, int n, const int32_t* d_target, int64_t n_target,
                      unsigned char** mask, double** rmag, int** rcol, double2** rval, void* base, cudaStream_t st) {
  unsigned char* p = (unsigned char*)base;
  auto take = [&](size_t b) {
    unsigned char* q = p;
    p += (b + 255) & ~size_t(255);
    return q;
  };
  *rval = (double2*)take(sizeof(double2) * n * batch);
  *rmag = (double*)take(sizeof(double) * n * batch);
  *rcol = (int*)take(sizeof(int) * n * batch);
  *mask = d_target ? (unsigned char*)take(n) : nullptr;
  if (d_target) {
    fill_mask_kernel<<<(n + 255) / 256, 256, 0, st>>>(*mask, n, d_target, (int)n_target);
    if (n_target > 0) set_mask_kernel<<<(int)((n_target + 255) / 256), 256, 0, st>>>(*mask, d_target, (int)n_target);
    note_launch(n_target > 0 ? 2 : 1);
  }
  dim3 grid((n + 7) / 8, (unsigned)batch);
  rowmax_init_kernel<<<grid, 256, 0, st>>>(d_h, n, *mask, d_target, (int)n_target, *rmag, *rcol, *rval);
  QCH_LAUNCH_CHECK("rowmax_init_kernel");
  note_launch(1);
  return QCH_OK;
}

static size_t npad_ws_bytes(int64_t batch, int n) {
  return 3 * 256 + (sizeof(double2) + sizeof(double) + sizeof(int)) * (size_t)n * batch + (size_t)n + 4 * 256 +
         sizeof(NpadJob) * batch;
}

// UnitarityDrift audit (npad.py:254-259)
extern "C" int qch_unitarity_defect_c128(const void* d_u, int64_t batch, int64_t n, double* d_defect, void* stream);

extern "C" int qch_npad_run_dense_c128(void* d_h, int64_t n, const int32_t* d_target, int64_t n_target,
                                       double threshold, int64_t max_iter, void* d_u, int32_t* d_pivots,
                                       int64_t pivot_cap, int64_t* applied, int* converged, void* stream) {
  if (n < 1) return fail(QCH_ERR_VALUE, "dimension must be at least 1");
  if (n >= 65536) return fail(QCH_ERR_UNSUPPORTED, "npad: dimension must be < 65536");
  cudaStream_t st = (cudaStream_t)stream;
  const int ni = (int)n;
  Workspace ws(st);
  QCH_CUDA(ws.alloc(npad_ws_bytes(1, ni) + 256));
  unsigned char* base = (unsigned char*)ws.p;
  int* d_flag = (int*)base;
  NpadJob* d_job = (NpadJob*)(base + 256);
  unsigned char* rest = base + 256 + ((sizeof(NpadJob) + 255) & ~size_t(255));
  int rc = qch_hermitian_exact_c128(d_h, n, d_flag, stream);
  if (rc) return rc;
  unsigned char* mask;
  double* rmag;
  int* rcol;
  double2* rval;
  rc = npad_setup((const double2*)d_h, 1, ni, d_target, n_target, &mask, &rmag, &rcol, &rval, rest, st);
  if (rc) return rc;
  int nonherm = 0;
  QCH_CUDA(cudaMemcpyAsync(&nonherm, d_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  QCH_CUDA(cudaStreamSynchronize(st));

  NpadJob job;
  job.h = (double2*)d_h;
  job.u = (double2*)d_u;
  job.rmag = rmag;
  job.rcol = rcol;
  job.rval = rval;
  job.pivots = d_pivots;
  job.pivot_cap = d_pivots ? pivot_cap : 0;
  job.threshold = threshold;
  job.applied = 0;
  job.status = 0;
  NpadCommon cm;
  cm.n = ni;
  cm.inT = mask;
  cm.tlist = d_target;
  cm.n_target = (int)n_target;
  cm.herm = nonherm ? 0 : 1;
  cm.max_iter = max_iter;
  int cpt, threads;
  npad_shape(ni, 1024, &cpt, &threads);
  cm.stage_h = npad_smem_bytes(ni, threads, true) <= (size_t)max_smem_optin() ? 1 : 0;
  const int64_t audit_every = 100;  // UNITARY_CHECK_EVERY, npad.py:216
  double* d_defect = nullptr;
  Workspace ws2(st);
  if (d_u) {
    QCH_CUDA(ws2.alloc(sizeof(double)));
    d_defect = (double*)ws2.p;
  }
  while (true) {
    cm.stop_at = d_u ? ((job.applied / audit_every) + 1) * audit_every : INT64_MAX;
    QCH_CUDA(cudaMemcpyAsync(d_job, &job, sizeof(NpadJob), cudaMemcpyHostToDevice, st));
    rc = npad_launch(d_job, 1, cm, 1024, st);
    if (rc) return rc;
    QCH_CUDA(cudaMemcpyAsync(&job, d_job, sizeof(NpadJob), cudaMemcpyDeviceToHost, st));
    QCH_CUDA(cudaStreamSynchronize(st));
    if (job.status != 2) break;
    // paused at a multiple of 100 rotations: audit ||UU^dag - I||_F <= 1e-10 N
    rc = qch_unitarity_defect_c128(d_u, 1, n, d_defect, stream);
    if (rc) return rc;
    double defect = 0.0;
    QCH_CUDA(cudaMemcpyAsync(&defect, d_defect, sizeof(double), cudaMemcpyDeviceToHost, st));
    QCH_CUDA(cudaStreamSynchronize(st));
    if (!(defect <= 1e-10 * (double)n)) {
      char buf[160];
      snprintf(buf, sizeof buf, "accumulated unitary drift %.3e after %lld rotations", defect, (long long)job.applied);
      return fail(QCH_ERR_UNITARITY_DRIFT, buf);
    }
  }
  *applied = job.applied;
  *converged = job.status == 0 ? 1 : 0;
  return QCH_OK;
}

__global__ void batch_jobs_kernel(NpadJob* jobs, double2* h, int64_t n, const double* thr, double* rmag, int* rcol,
                                  double2* rval, int64_t batch) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= batch) return;
  NpadJob j;
  j.h = h + b * n * n;
  j.u = nullptr;
  j.rmag = rmag + b * n;
  j.rcol = rcol + b * n;
  j.rval = rval + b * n;
  j.pivots = nullptr;
  j.pivot_cap = 0;
  j.threshold = thr[b];
  j.applied = 0;
  j.status = 0;
  jobs[b] = j;
}
__global__ void batch_out_kernel(const NpadJob* jobs, int64_t batch, int64_t* applied, int32_t* conv) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= batch) return;
  applied[b] = jobs[b].applied;
  conv[b] = jobs[b].status == 0 ? 1 : 0;
}

extern "C" int qch_npad_run_batch_c128(void* d_h, int64_t batch, int64_t n, const int32_t* d_target,
                                       int64_t n_target, const double* d_thresholds, int64_t max_iter,
                                       int64_t* d_applied, int32_t* d_converged, void* stream) {
  if (batch <= 0) return QCH_OK;
  if (n < 1) return fail(QCH_ERR_VALUE, "dimension must be at least 1");
  if (n >= 65536) return fail(QCH_ERR_UNSUPPORTED, "npad: dimension must be < 65536");
  cudaStream_t st = (cudaStream_t)stream;
  const int ni = (int)n;
  Workspace ws(st);
  QCH_CUDA(ws.alloc(npad_ws_bytes(batch, ni) + 256));
  NpadJob* d_jobs = (NpadJob*)ws.p;
  unsigned char* rest = (unsigned char*)ws.p + ((sizeof(NpadJob) * batch + 255) & ~size_t(255));
  unsigned char* mask;
  double* rmag;
  int* rcol;
  double2* rval;
  int rc = npad_setup((const double2*)d_h, batch, ni, d_target, n_target, &mask, &rmag, &rcol, &rval, rest, st);
  if (rc) return rc;
  batch_jobs_kernel<<<(int)((batch + 127) / 128), 128, 0, st>>>(d_jobs, (double2*)d_h, n, d_thresholds, rmag, rcol,
                                                                   rval, batch);
  note_launch(1);
  NpadCommon cm;
  cm.n = ni;
  cm.inT = mask;
  cm.tlist = d_target;
  cm.n_target = (int)n_target;
  cm.herm = 1;
  cm.max_iter = max_iter;
  cm.stop_at = INT64_MAX;
  int cpt, threads;
  npad_shape(ni, 256, &cpt, &threads);
  cm.stage_h = 0;
  rc = npad_launch(d_jobs, (int)batch, cm, 256, st);
  if (rc) return rc;
  batch_out_kernel<<<(int)((batch + 127) / 128), 128, 0, st>>>(d_jobs, batch, d_applied, d_converged);
  note_launch(1);
  QCH_LAUNCH_CHECK("batch_out_kernel");
  return QCH_OK;
}
