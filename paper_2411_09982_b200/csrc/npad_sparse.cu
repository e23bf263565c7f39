// npad_sparse.cu — the sparse Givens rotation of NPAD on a device CSR:
// _conjugate_sparse (npad.py:148-232), i.e. H <- U H U^dag for a rotation in
// the (i, j) plane, producing a NEW CSR (operators are immutable,
// operators.py:43-57).  The paper's headline NPAD benchmark is one such
// rotation on the sparse ladder a^dag a + (a + a^dag) at N = 1e5..1e8
// (experiments.py:420-453).
//
// Only rows/columns i, j change, so the new CSR is the old one with a handful
// of rows rewritten and every other row SHIFTED by the nnz change of the
// rewritten rows before it.  The pipeline is one O(1)-sized piece of work
// plus three streaming passes (HBM-bound):
//   pair     (1 thread)  merge rows i, j into the new rows i, j with the
//                        reference's arithmetic (np.add.at order, the three
//                        corner formulas in scalar (non-FMA) complex math,
//                        fill-in below 1e-15 max|H| dropped);
//   classify (thread/row) rows x != i, j holding or gaining an entry in
//                        column i or j -> "changed", with their nnz change;
//   sort     (1 block)   changed rows by index, prefix sums of the changes;
//   indptr   (thread/row) new_indptr[x] = old_indptr[x] + sum of changes of
//                        changed rows before x (binary search);
//   copy     (thread/nnz) unchanged rows' entries to their shifted slots;
//   rows     (warp/changed row) the rewritten rows.
// Bit-identical to the reference (tests/golden/npad_sparse.npz).
#include <algorithm>
#include <cstring>

#include "qch_internal.h"
#include "qch_math.cuh"

namespace qch {
namespace {

constexpr int kMaxChanged = 1 << 16;  // changed rows handled per rotation

// scalar complex multiply as CPython / numpy scalar math do it (no FMA)
__device__ __forceinline__ cplx cmul_scalar(cplx a, cplx b) {
  return mkc(QSUB(QMUL(a.re, b.re), QMUL(a.im, b.im)), QADD(QMUL(a.re, b.im), QMUL(a.im, b.re)));
}

struct PairOut {
  int64_t la, lb;     // lengths of the new rows i, j
  int64_t nchanged;   // rows in the changed list (incl. i, j)
  int64_t nnz_out;
  int overflow;
};

struct SpArgs {
  const int64_t* indptr;
  const int32_t* indices;
  const double2* data;
  int64_t n, nnz;
  int i, j;
  double c;
  double2 s;      // block s = -sin_half * e^{i phase}
  double drop;    // 1e-15 * max|H|
  // scratch
  int32_t* a_col;
  double2* a_val;
  int32_t* b_col;
  double2* b_val;
  int64_t cap_ab;
  int32_t* chg_row;  // changed rows (unsorted, then sorted)
  int64_t* chg_delta;
  int64_t* chg_pref;  // exclusive prefix of deltas (sorted order)
  int64_t* chg_end;   // old_indptr[r + 1] (sorted order)
  unsigned long long* counter;
  PairOut* po;
  // output
  int64_t* out_indptr;
  int32_t* out_indices;
  double2* out_data;
};

__device__ __forceinline__ int64_t find_col(const int32_t* cols, int64_t len, int32_t c) {
  int64_t lo = 0, hi = len;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (cols[mid] < c) lo = mid + 1;
    else hi = mid;
  }
  return (lo < len && cols[lo] == c) ? lo : -1;
}

// (x, value) setter on a sorted list with insertion (npad.py:170-175)
__device__ void set_at(int32_t* cols, double2* vals, int64_t& len, int32_t k, double2 v) {
  int64_t pos = 0;
  while (pos < len && cols[pos] < k) ++pos;
  if (pos < len && cols[pos] == k) {
    vals[pos] = v;
    return;
  }
  for (int64_t q = len; q > pos; --q) {
    cols[q] = cols[q - 1];
    vals[q] = vals[q - 1];
  }
  cols[pos] = k;
  vals[pos] = v;
  ++len;
}

__global__ void pair_kernel(SpArgs g) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int i = g.i, j = g.j;
  const int64_t i0 = g.indptr[i], i1 = g.indptr[i + 1], j0 = g.indptr[j], j1 = g.indptr[j + 1];
  const cplx s = d2c(g.s), sc = cconj(s), msc = mkc(-sc.re, -sc.im);
  const cplx cw = mkc(g.c, 0.0);
  // _row_combination (npad.py:148-159): acc = 0 + wi*vi (+ wj*vj), in
  // ascending column order; ufunc multiplies use numpy's FMA pattern
  int64_t la = 0, lb = 0;
  int64_t p = i0, q = j0;
  while (p < i1 || q < j1) {
    const int32_t ci = p < i1 ? g.indices[p] : INT32_MAX;
    const int32_t cj = q < j1 ? g.indices[q] : INT32_MAX;
    const int32_t col = min(ci, cj);
    cplx a = mkc(0.0, 0.0), b = mkc(0.0, 0.0);
    if (ci == col) {
      const cplx vi = d2c(g.data[p++]);
      a = cadd(a, np_cmul(cw, vi));
      b = cadd(b, np_cmul(s, vi));
    }
    if (cj == col) {
      const cplx vj = d2c(g.data[q++]);
      a = cadd(a, np_cmul(msc, vj));
      b = cadd(b, np_cmul(cw, vj));
    }
    if (la + 2 >= g.cap_ab) {
      g.po->overflow = 1;
      return;
    }
    g.a_col[la] = col;
    g.a_val[la++] = c2d(a);
    g.b_col[lb] = col;
    g.b_val[lb++] = c2d(b);
  }
  // right factor on columns i, j (npad.py:188-197) in Python/numpy scalar math
  auto get = [&](const int32_t* cols, const double2* vals, int64_t len, int32_t k) {
    const int64_t pos = find_col(cols, len, k);
    return pos >= 0 ? d2c(vals[pos]) : mkc(0.0, 0.0);
  };
  const cplx ai = get(g.a_col, g.a_val, la, i), aj = get(g.a_col, g.a_val, la, j);
  const cplx bi = get(g.b_col, g.b_val, lb, i), bj = get(g.b_col, g.b_val, lb, j);
  const cplx cai = mkc(QMUL(g.c, ai.re), QMUL(g.c, ai.im));  // Python float * complex
  const cplx caj = mkc(QMUL(g.c, aj.re), QMUL(g.c, aj.im));
  const cplx cbj = mkc(QMUL(g.c, bj.re), QMUL(g.c, bj.im));
  const double new_ai = QSUB(cai.re, cmul_scalar(s, aj).re);
  const cplx new_aj = cadd(cmul_scalar(sc, ai), caj);
  const double new_bj = QADD(cmul_scalar(sc, bi).re, cbj.re);
  set_at(g.a_col, g.a_val, la, i, make_double2(new_ai, 0.0));
  set_at(g.a_col, g.a_val, la, j, c2d(new_aj));
  set_at(g.b_col, g.b_val, lb, i, c2d(cconj(new_aj)));
  set_at(g.b_col, g.b_val, lb, j, make_double2(new_bj, 0.0));
  // drop fill-in below the threshold (npad.py:199-204): |v| (numpy) > drop
  int64_t ka = 0, kb = 0;
  for (int64_t k = 0; k < la; ++k)
    if (np_cabs(g.a_val[k].x, g.a_val[k].y) > g.drop) {
      g.a_col[ka] = g.a_col[k];
      g.a_val[ka++] = g.a_val[k];
    }
  for (int64_t k = 0; k < lb; ++k)
    if (np_cabs(g.b_val[k].x, g.b_val[k].y) > g.drop) {
      g.b_col[kb] = g.b_col[k];
      g.b_val[kb++] = g.b_val[k];
    }
  g.po->la = ka;
  g.po->lb = kb;
  // rows i and j head the changed list
  g.chg_row[0] = i;
  g.chg_delta[0] = ka - (i1 - i0);
  g.chg_row[1] = j;
  g.chg_delta[1] = kb - (j1 - j0);
  *g.counter = 2;
}

// rows x != i, j: entries in columns i / j now and after the rotation.
// kClassU rows per thread with their loads issued together (each row costs
// two dependent loads: indptr, then its first / last column); a row is
// searched only when its column range can hold i or j, or x can be a column
// of the new rows i, j.
constexpr int kClassU = 4;
__device__ __forceinline__ void classify_row(const SpArgs& g, int64_t x, int64_t r0, int64_t r1, int32_t cfirst,
                                             int32_t clast, int32_t lo_ij, int32_t hi_ij, int32_t amin, int32_t amax) {
  if (x == g.i || x == g.j) return;
  int old_cnt = 0;
  if (r1 > r0 && cfirst <= hi_ij && clast >= lo_ij)
    old_cnt = (find_col(g.indices + r0, r1 - r0, g.i) >= 0) + (find_col(g.indices + r0, r1 - r0, g.j) >= 0);
  int new_cnt = 0;
  if (x >= amin && x <= amax) {
    const int64_t la = g.po->la, lb = g.po->lb;
    new_cnt = (find_col(g.a_col, la, (int32_t)x) >= 0) + (find_col(g.b_col, lb, (int32_t)x) >= 0);
  }
  if (old_cnt == 0 && new_cnt == 0) return;
  const unsigned long long k = atomicAdd(g.counter, 1ull);
  if (k >= (unsigned long long)kMaxChanged) {
    g.po->overflow = 1;
    return;
  }
  g.chg_row[k] = (int32_t)x;
  g.chg_delta[k] = new_cnt - old_cnt;
}
__global__ void classify_kernel(SpArgs g) {
  const int32_t lo_ij = min(g.i, g.j), hi_ij = max(g.i, g.j);
  // column range of the new rows i, j (sorted lists)
  const int64_t la = g.po->la, lb = g.po->lb;
  int32_t amin = 0x7fffffff, amax = -1;
  if (la > 0) {
    amin = min(amin, g.a_col[0]);
    amax = max(amax, g.a_col[la - 1]);
  }
  if (lb > 0) {
    amin = min(amin, g.b_col[0]);
    amax = max(amax, g.b_col[lb - 1]);
  }
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; base < g.n; base += nth * kClassU) {
    int64_t r0[kClassU], r1[kClassU];
    int32_t cf[kClassU], cl[kClassU];
#pragma unroll
    for (int u = 0; u < kClassU; ++u) {
      const int64_t x = base + u * nth;
      r0[u] = x < g.n ? g.indptr[x] : 0;
      r1[u] = x < g.n ? g.indptr[x + 1] : 0;
    }
#pragma unroll
    for (int u = 0; u < kClassU; ++u) {
      cf[u] = r1[u] > r0[u] ? g.indices[r0[u]] : 0;
      cl[u] = r1[u] > r0[u] ? g.indices[r1[u] - 1] : -1;
    }
#pragma unroll
    for (int u = 0; u < kClassU; ++u) {
      const int64_t x = base + u * nth;
      if (x < g.n) classify_row(g, x, r0[u], r1[u], cf[u], cl[u], lo_ij, hi_ij, amin, amax);
    }
  }
}

// sort the changed rows, prefix sums of the nnz changes, total
__global__ void sort_changed_kernel(SpArgs g) {
  __shared__ int64_t s_n;
  if (threadIdx.x == 0) {
    const unsigned long long cnt = *g.counter;
    s_n = (int64_t)(cnt < (unsigned long long)kMaxChanged ? cnt : (unsigned long long)kMaxChanged);
  }
  __syncthreads();
  const int64_t m = s_n;
  // odd-even transposition sort (the list is tiny for sparse NPAD)
  for (int64_t pass = 0; pass < m; ++pass) {
    for (int64_t k = 2 * threadIdx.x + (pass & 1); k + 1 < m; k += 2 * blockDim.x) {
      if (g.chg_row[k] > g.chg_row[k + 1]) {
        const int32_t r = g.chg_row[k];
        g.chg_row[k] = g.chg_row[k + 1];
        g.chg_row[k + 1] = r;
        const int64_t d = g.chg_delta[k];
        g.chg_delta[k] = g.chg_delta[k + 1];
        g.chg_delta[k + 1] = d;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int64_t k = 0; k < m; ++k) {
      g.chg_pref[k] = acc;
      acc += g.chg_delta[k];
      g.chg_end[k] = g.indptr[g.chg_row[k] + 1];
    }
    g.po->nchanged = m;
    g.po->nnz_out = g.nnz + acc;
  }
}

// number of changed rows r < x (sorted list)
__device__ __forceinline__ int64_t changed_before(const int32_t* rows, int64_t m, int64_t x) {
  int64_t lo = 0, hi = m;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (rows[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void indptr_kernel(SpArgs g) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x > g.n) return;
  const int64_t m = g.po->nchanged;
  const int64_t k = changed_before(g.chg_row, m, x);
  const int64_t shift = (k == 0) ? 0 : g.chg_pref[k - 1] + g.chg_delta[k - 1];
  g.out_indptr[x] = g.indptr[x] + shift;
}

// entries of unchanged rows to their shifted slots (coalesced both ways).
// A warp moves chunks of 32 x kCopyU consecutive entries; the few changed
// rows split the CSR into segments of constant shift, so a chunk that does
// not touch a changed row (nearly all of them) is moved with one shift and
// kCopyU independent loads in flight per lane; a chunk that does falls back
// to the per-entry lookup.
constexpr int kCopyU = 8;
__device__ __forceinline__ int64_t seg_of(const SpArgs& g, int64_t m, int64_t e) {
  int64_t lo = 0, hi = m;  // changed rows whose old range ends at or before e
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (g.chg_end[mid] <= e) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
__global__ void copy_kernel(SpArgs g) {
  const int64_t m = g.po->nchanged;
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int64_t kChunk = 32 * kCopyU;
  for (int64_t base = w * kChunk; base < g.nnz; base += nw * kChunk) {
    const int64_t end = base + kChunk < g.nnz ? base + kChunk : g.nnz;
    const int64_t lo = seg_of(g, m, base);
    // the next changed row's old start: the chunk is uniform if it ends before it
    const bool uniform = lo == m || g.indptr[g.chg_row[lo]] >= end;
    if (uniform) {
      const int64_t shift = (lo == 0) ? 0 : g.chg_pref[lo - 1] + g.chg_delta[lo - 1];
      int32_t ci[kCopyU];
      double2 cv[kCopyU];
#pragma unroll
      for (int k = 0; k < kCopyU; ++k) {
        const int64_t e = base + k * 32 + lane;
        if (e < end) {
          ci[k] = g.indices[e];
          cv[k] = g.data[e];
        }
      }
#pragma unroll
      for (int k = 0; k < kCopyU; ++k) {
        const int64_t e = base + k * 32 + lane;
        if (e < end) {
          g.out_indices[e + shift] = ci[k];
          g.out_data[e + shift] = cv[k];
        }
      }
    } else {
      for (int64_t e = base + lane; e < end; e += 32) {
        const int64_t l2 = seg_of(g, m, e);
        if (l2 < m && g.indptr[g.chg_row[l2]] <= e) continue;  // inside changed row chg_row[l2]: rows_kernel
        const int64_t shift = (l2 == 0) ? 0 : g.chg_pref[l2 - 1] + g.chg_delta[l2 - 1];
        g.out_indices[e + shift] = g.indices[e];
        g.out_data[e + shift] = g.data[e];
      }
    }
  }
}

// the changed rows: i, j = the new rows; others = old entries without
// columns i, j, plus (x, i) = conj(new a[x]) and (x, j) = conj(new b[x])
__global__ void rows_kernel(SpArgs g) {
  const int64_t m = g.po->nchanged;
  const int64_t la = g.po->la, lb = g.po->lb;
  for (int64_t k = blockIdx.x; k < m; k += gridDim.x) {
    if (threadIdx.x != 0) continue;
    const int32_t x = g.chg_row[k];
    int64_t o = g.out_indptr[x];
    if (x == g.i) {
      for (int64_t q = 0; q < la; ++q, ++o) {
        g.out_indices[o] = g.a_col[q];
        g.out_data[o] = g.a_val[q];
      }
      continue;
    }
    if (x == g.j) {
      for (int64_t q = 0; q < lb; ++q, ++o) {
        g.out_indices[o] = g.b_col[q];
        g.out_data[o] = g.b_val[q];
      }
      continue;
    }
    const int64_t pa = find_col(g.a_col, la, x), pb = find_col(g.b_col, lb, x);
    const int64_t r0 = g.indptr[x], r1 = g.indptr[x + 1];
    // merge: old entries (minus cols i, j) with the new (x, i), (x, j), ascending
    int32_t ins_c[2];
    double2 ins_v[2];
    int nins = 0;
    if (pa >= 0) {
      ins_c[nins] = g.i;
      ins_v[nins++] = make_double2(g.a_val[pa].x, -g.a_val[pa].y);
    }
    if (pb >= 0) {
      ins_c[nins] = g.j;
      ins_v[nins++] = make_double2(g.b_val[pb].x, -g.b_val[pb].y);
    }
    int q = 0;
    for (int64_t e = r0; e < r1; ++e) {
      const int32_t col = g.indices[e];
      while (q < nins && ins_c[q] < col) {
        g.out_indices[o] = ins_c[q];
        g.out_data[o++] = ins_v[q++];
      }
      if (col == g.i || col == g.j) continue;
      g.out_indices[o] = col;
      g.out_data[o++] = g.data[e];
    }
    while (q < nins) {
      g.out_indices[o] = ins_c[q];
      g.out_data[o++] = ins_v[q++];
    }
  }
}

}  // namespace
}  // namespace qch

using namespace qch;

// _conjugate_sparse (npad.py:178-232) on a device CSR (sorted column indices,
// no explicit zeros; indptr int64, indices int32, data complex128).  Writes
// the new CSR into d_out_* (capacity out_cap entries; the new nnz is at most
// nnz + 4 * (len(row i) + len(row j)) + 8) and its nnz to *nnz_out (host).
// Synchronous.  Rotation = _block_params (npad.py:126-128): cos_half and
// s = -sin_half e^{i phase} (formed by the caller exactly as the reference
// does, so the arithmetic here is bit-identical); max_abs = max|H| of the
// input (the drop threshold is 1e-15 * max_abs).
extern "C" int qch_npad_sparse_rotate_c128(const int64_t* d_indptr, const int32_t* d_indices, const void* d_data,
                                           int64_t n, int64_t nnz, int64_t i, int64_t j, double cos_half,
                                           double s_re, double s_im, double max_abs, int64_t* d_out_indptr,
                                           int32_t* d_out_indices, void* d_out_data, int64_t out_cap,
                                           int64_t* nnz_out, void* stream) {
  if (!(0 <= i && i < j && j < n)) return fail(QCH_ERR_INDEX, "need 0 <= i < j < n");
  if (n >= INT32_MAX) return fail(QCH_ERR_UNSUPPORTED, "sparse rotation: n must fit int32 column indices");
  cudaStream_t st = (cudaStream_t)stream;
  int64_t ends[4];
  QCH_CUDA(cudaMemcpyAsync(ends, d_indptr + i, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  QCH_CUDA(cudaMemcpyAsync(ends + 2, d_indptr + j, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  QCH_CUDA(cudaStreamSynchronize(st));
  const int64_t li = ends[1] - ends[0], lj = ends[3] - ends[2];
  const int64_t cap_ab = li + lj + 4;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t bytes = 2 * al(sizeof(int32_t) * cap_ab) + 2 * al(sizeof(double2) * cap_ab) +
                       al(sizeof(int32_t) * kMaxChanged) + 3 * al(sizeof(int64_t) * kMaxChanged) + al(64) +
                       al(sizeof(PairOut));
  void* ws = nullptr;
  ensure_pool();
  QCH_CUDA(cudaMallocAsync(&ws, bytes, st));
  unsigned char* p = (unsigned char*)ws;
  auto take = [&](size_t b) {
    unsigned char* q = p;
    p += al(b);
    return q;
  };
  SpArgs g;
  g.indptr = d_indptr;
  g.indices = d_indices;
  g.data = (const double2*)d_data;
  g.n = n;
  g.nnz = nnz;
  g.i = (int)i;
  g.j = (int)j;
  g.c = cos_half;
  g.s = make_double2(s_re, s_im);
  g.drop = 1e-15 * max_abs;
  g.cap_ab = cap_ab;
  g.a_col = (int32_t*)take(sizeof(int32_t) * cap_ab);
  g.b_col = (int32_t*)take(sizeof(int32_t) * cap_ab);
  g.a_val = (double2*)take(sizeof(double2) * cap_ab);
  g.b_val = (double2*)take(sizeof(double2) * cap_ab);
  g.chg_row = (int32_t*)take(sizeof(int32_t) * kMaxChanged);
  g.chg_delta = (int64_t*)take(sizeof(int64_t) * kMaxChanged);
  g.chg_pref = (int64_t*)take(sizeof(int64_t) * kMaxChanged);
  g.chg_end = (int64_t*)take(sizeof(int64_t) * kMaxChanged);
  g.counter = (unsigned long long*)take(64);
  g.po = (PairOut*)take(sizeof(PairOut));
  g.out_indptr = d_out_indptr;
  g.out_indices = d_out_indices;
  g.out_data = (double2*)d_out_data;
  QCH_CUDA(cudaMemsetAsync(g.po, 0, sizeof(PairOut), st));
  void* pr = prof_begin("npad_sparse_rotate", st);
  pair_kernel<<<1, 32, 0, st>>>(g);
  classify_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 256 * kClassU - 1) / (256 * kClassU),
                                                                        (int64_t)sm_count() * 32)),
                    256, 0, st>>>(g);
  sort_changed_kernel<<<1, 256, 0, st>>>(g);
  QCH_LAUNCH_CHECK("sparse rotate (pair/classify/sort)");
  PairOut po;
  QCH_CUDA(cudaMemcpyAsync(&po, g.po, sizeof po, cudaMemcpyDeviceToHost, st));
  QCH_CUDA(cudaStreamSynchronize(st));
  if (po.overflow) {
    prof_end(pr, st);
    cudaFreeAsync(ws, st);
    return fail(QCH_ERR_UNSUPPORTED, "sparse rotation: more changed rows than supported");
  }
  if (po.nnz_out > out_cap) {
    prof_end(pr, st);
    cudaFreeAsync(ws, st);
    return fail(QCH_ERR_VALUE, "sparse rotation: output capacity too small");
  }
  void* pr2 = prof_begin("npad_sparse_stream", st);  // the two HBM-streaming passes
  indptr_kernel<<<(unsigned)((n + 1 + 255) / 256), 256, 0, st>>>(g);
  const int blocks = (int)std::min<int64_t>((nnz + 255) / 256, (int64_t)sm_count() * 16);
  if (nnz > 0) copy_kernel<<<std::max(1, blocks), 256, 0, st>>>(g);
  prof_end(pr2, st);
  rows_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(po.nchanged, 4096)), 32, 0, st>>>(g);
  prof_end(pr, st);
  QCH_LAUNCH_CHECK("sparse rotate (indptr/copy/rows)");
  note_launch(6);
  QCH_CUDA(cudaFreeAsync(ws, st));
  QCH_CUDA(cudaStreamSynchronize(st));
  *nnz_out = po.nnz_out;
  return QCH_OK;
}

// HermitianOperator.entry on a device CSR (operators.py:101-102): the values
// at (j, i), (i, i), (j, j) — what givens_rotation_matrix reads
// (npad.py:111-117).  d_out: 3 complex (device).
__global__ void sparse_entries_kernel(const int64_t* indptr, const int32_t* indices, const double2* data, int i,
                                      int j, double2* out) {
  const int t = threadIdx.x;
  if (t >= 3) return;
  const int r = (t == 0) ? j : (t == 1 ? i : j);
  const int c = (t == 0) ? i : (t == 1 ? i : j);
  const int64_t r0 = indptr[r], r1 = indptr[r + 1];
  const int64_t pos = find_col(indices + r0, r1 - r0, c);
  out[t] = pos >= 0 ? data[r0 + pos] : make_double2(0.0, 0.0);
}

extern "C" int qch_npad_sparse_entries_c128(const int64_t* d_indptr, const int32_t* d_indices, const void* d_data,
                                            int64_t n, int64_t i, int64_t j, void* d_out, void* stream) {
  if (!(0 <= i && i < n && 0 <= j && j < n)) return fail(QCH_ERR_INDEX, "index out of range");
  sparse_entries_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(d_indptr, d_indices, (const double2*)d_data, (int)i,
                                                            (int)j, (double2*)d_out);
  QCH_LAUNCH_CHECK("sparse_entries_kernel");
  note_launch(1);
  return QCH_OK;
}

// the ladder benchmark operator a^dag a + (a + a^dag) on n Fock states
// (models.py:194-209) built directly as a device CSR as HermitianOperator
// stores it (explicit zeros eliminated, operators.py:48-53): row 0 holds
// column 1 (its diagonal is 0), row r >= 1 holds columns r-1, r, r+1 with
// sqrt(r), r, sqrt(r+1).  d_indptr (n+1), d_indices / d_data (3n - 3).
__global__ void ladder_csr_kernel(int64_t n, int64_t* indptr, int32_t* indices, double2* data) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r > n) return;
  indptr[r] = (r == 0) ? 0 : (r == n ? 3 * n - 3 : 3 * r - 2);
  if (r == n) return;
  if (r == 0) {
    indices[0] = 1;
    data[0] = make_double2(1.0, 0.0);
    return;
  }
  int64_t o = 3 * r - 2;
  indices[o] = (int32_t)(r - 1);
  data[o++] = make_double2(sqrt((double)r), 0.0);
  indices[o] = (int32_t)r;
  data[o++] = make_double2((double)r, 0.0);
  if (r + 1 < n) {
    indices[o] = (int32_t)(r + 1);
    data[o] = make_double2(sqrt((double)(r + 1)), 0.0);
  }
}

extern "C" int qch_build_ladder_csr_c128(int64_t n, int64_t* d_indptr, int32_t* d_indices, void* d_data,
                                         void* stream) {
  if (n < 2 || n >= INT32_MAX) return fail(QCH_ERR_VALUE, "ladder: need 2 <= n < 2^31");
  ladder_csr_kernel<<<(unsigned)((n + 1 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, d_indptr, d_indices,
                                                                                        (double2*)d_data);
  QCH_LAUNCH_CHECK("ladder_csr_kernel");
  note_launch(1);
  return QCH_OK;
}

// ---------------------------------------------------------------------------
// _largest_relevant (npad.py:300-317) on a device CSR: the strict-lower-
// triangle entry of largest numpy |z| (subspace mode: exactly one endpoint in
// the target), ties to the smallest (c, r).  Thread per row, block argmax,
// then one block over the block winners.
#include "npad_select.cuh"

namespace qch {
namespace {

constexpr int kSelThreads = 256;

__device__ __forceinline__ Cand sel_shfl(const Cand& c, int src) {
  Cand o;
  o.q = __shfl_sync(kFull, c.q, src);
  o.m = __shfl_sync(kFull, c.m, src);
  o.cr = __shfl_sync(kFull, c.cr, src);
  o.v.x = __shfl_sync(kFull, c.v.x, src);
  o.v.y = __shfl_sync(kFull, c.v.y, src);
  return o;
}

__device__ Cand sel_block_best(Cand c) {
  __shared__ Cand s_w[kSelThreads / 32];
  const int wl = warp_argmax(c);
  const Cand w = (wl >= 0) ? sel_shfl(c, wl) : cand_none();
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = w;
  __syncthreads();
  Cand b = s_w[0];
  for (int k = 1; k < kSelThreads / 32; ++k) cand_take(b, s_w[k]);
  __syncthreads();
  return b;
}

__global__ void sparse_select_kernel(const int64_t* indptr, const int32_t* indices, const double2* data, int64_t n,
                                     const unsigned char* inT, int ek, Cand* part) {
  Cand best = cand_none();
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r < n) {
    for (int64_t e = indptr[r]; e < indptr[r + 1]; ++e) {
      const int c = indices[e];
      if (c >= r) break;  // sorted: the strict lower part comes first
      if (inT != nullptr && inT[c] == inT[r]) continue;
      const double2 v = data[e];
      if (v.x == 0.0 && v.y == 0.0) continue;
      cand_take(best, make_cand(v, ((unsigned)c << 16) | (unsigned)r, ek != 0));
    }
  }
  const Cand b = sel_block_best(best);
  if (threadIdx.x == 0) part[blockIdx.x] = b;
}

__global__ void sparse_select_final_kernel(const Cand* part, int64_t nparts, double* out) {
  Cand best = cand_none();
  for (int64_t k = threadIdx.x; k < nparts; k += blockDim.x) cand_take(best, part[k]);
  const Cand b = sel_block_best(best);
  if (threadIdx.x == 0) {
    out[0] = (b.q > 0.0) ? (double)(b.cr >> 16) : -1.0;
    out[1] = (b.q > 0.0) ? (double)(b.cr & 0xffffu) : -1.0;
    out[2] = (b.q > 0.0) ? np_cabs(b.v.x, b.v.y) : 0.0;
  }
}

}  // namespace
}  // namespace qch

// (i, j, |H[j, i]|) of the largest relevant coupling of a device CSR
// (npad.py:300-317); i = j = -1 when there is none.  d_mask: n bytes, 1 for
// target levels (null: full mode).  Synchronous; result in host out[3].
// Indices must be < 65536 (the packed tie-break key).
extern "C" int qch_npad_sparse_select_c128(const int64_t* d_indptr, const int32_t* d_indices, const void* d_data,
                                           int64_t n, const unsigned char* d_mask, int exact_keys, double* out,
                                           void* stream) {
  if (n >= 65536) return fail(QCH_ERR_UNSUPPORTED, "sparse npad_run: dimension must be < 65536");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t blocks = (n + kSelThreads - 1) / kSelThreads;
  void* ws = nullptr;
  ensure_pool();
  QCH_CUDA(cudaMallocAsync(&ws, sizeof(Cand) * blocks + 64, st));
  Cand* part = (Cand*)ws;
  double* d_out = (double*)(part + blocks);
  sparse_select_kernel<<<(unsigned)std::max<int64_t>(1, blocks), kSelThreads, 0, st>>>(
      d_indptr, d_indices, (const double2*)d_data, n, d_mask, exact_keys, part);
  sparse_select_final_kernel<<<1, kSelThreads, 0, st>>>(part, std::max<int64_t>(1, blocks), d_out);
  QCH_LAUNCH_CHECK("sparse_select_kernel");
  note_launch(2);
  QCH_CUDA(cudaMemcpyAsync(out, d_out, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
  QCH_CUDA(cudaFreeAsync(ws, st));
  QCH_CUDA(cudaStreamSynchronize(st));
  return QCH_OK;
}
