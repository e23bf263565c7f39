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
#include <cstdlib>
#include <cstring>

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
  h += blockIdx.y * n;  // batched: grid.y = item, n elements each
  out += blockIdx.y;
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

// Hermiticity of a dense matrix, 32x32 tile pairs (R >= C) through shared
// memory so both the tile and its mirror are read coalesced: *flag |= 1 when
// some H[x,y] != conj(H[y,x]) (exact), and *defect (u64 bits of a
// non-negative double, atomicMax) = max |H[x,y] - conj(H[y,x])| with numpy's
// |z| (operators.py:104-116: max(abs(H - H^dag))).
__global__ void __launch_bounds__(256) hermitian_tiles_kernel(const double2* __restrict__ h, int64_t n, int* flag,
                                                              unsigned long long* defect) {
  __shared__ double2 ta[32][33], tb[32][33];
  // tile pair from the linear block index: row R, col C <= R
  const int t = blockIdx.x;
  int R = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((R + 1) * (R + 2) / 2 <= t) ++R;
  while (R * (R + 1) / 2 > t) --R;
  const int C = t - R * (R + 1) / 2;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int yy = ty; yy < 32; yy += 8) {
    const int64_t r = (int64_t)R * 32 + yy, c = (int64_t)C * 32 + tx;
    ta[yy][tx] = (r < n && c < n) ? h[r * n + c] : make_double2(0.0, 0.0);
    const int64_t r2 = (int64_t)C * 32 + yy, c2 = (int64_t)R * 32 + tx;
    tb[yy][tx] = (r2 < n && c2 < n) ? h[r2 * n + c2] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  int bad = 0;
  double worst = 0.0;
  for (int yy = ty; yy < 32; yy += 8) {
    const double2 a = ta[yy][tx], b = tb[tx][yy];  // H[r, c] and H[c, r]
    if (!(a.x == b.x && a.y == -b.y)) bad = 1;
    worst = fmax(worst, np_cabs(a.x - b.x, a.y + b.y));
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0 && flag) atomicOr(flag, 1);
  if (defect) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, off));
    if ((threadIdx.x & 31) == 0 && worst > 0.0) atomicMax(defect, (unsigned long long)__double_as_longlong(worst));
  }
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
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h != nullptr && x < n;
       x += (int64_t)gridDim.x * blockDim.x) {
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

__global__ void fill_mask_kernel(unsigned char* mask, int n, const int* tlist, int nt) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) mask[x] = 0;
}
__global__ void set_mask_kernel(unsigned char* mask, const int* tlist, int nt) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nt; q += gridDim.x * blockDim.x) mask[tlist[q]] = 1;
}

// ----------------------------------------------------------------------------
// transmon (x) resonator builder
__global__ void __launch_bounds__(256) build_tr_kernel(double2* __restrict__ h, int nq, int nr,
                                                       const double* __restrict__ prm,
                                                       unsigned long long* __restrict__ maxabs) {
  // block (x, item): rows r = x, x + gridDim.x, ...  A row holds at most 5
  // nonzeros (the diagonal and the couplings (q1 +- 1, k1 +- 1)): the block
  // streams the row's zeros with 16-byte stores (no index math), then one
  // thread per nonzero writes it — same values and order of operations as
  // the host builder, written once.
  const int n = nq * nr;
  const int64_t b = blockIdx.y;
  const double wq = prm[4 * b], al = prm[4 * b + 1], wr = prm[4 * b + 2], g = prm[4 * b + 3];
  double2* hb = h + b * (int64_t)n * n;
  double m = 0.0;
  for (int r = blockIdx.x; r < n; r += gridDim.x) {
    const int q1 = r / nr, k1 = r - q1 * nr;
    double2* row = hb + (int64_t)r * n;
    for (int c = threadIdx.x; c < n; c += blockDim.x) row[c] = make_double2(0.0, 0.0);
    __syncthreads();  // zeros before the nonzeros (different threads)
    const int t = threadIdx.x;
    if (t == 0) {
      // host builder (models.transmon_resonator_hamiltonian): n = b^dag b has
      // diagonal sqrt(q)^2 (not exactly q), a^dag a likewise; same op order.
      const double sq = sqrt((double)q1), sk = sqrt((double)k1);
      const double nn = QMUL(sq, sq), kk = QMUL(sk, sk);
      const double hq = QADD(QMUL(wq, nn), QMUL(QMUL(0.5, al), QMUL(nn, QSUB(nn, 1.0))));
      const double v = QADD(hq, QMUL(wr, kk));
      row[r] = make_double2(v, 0.0);
      m = fmax(m, fabs(v));  // numpy |v + 0j| = |v|
    } else if (t <= 4) {
      const int q2 = q1 + ((t & 1) ? 1 : -1), k2 = k1 + ((t & 2) ? 1 : -1);
      if (q2 >= 0 && q2 < nq && k2 >= 0 && k2 < nr) {
        const double bq = sqrt((double)(q1 > q2 ? q1 : q2));
        const double ak = sqrt((double)(k1 > k2 ? k1 : k2));
        const double v = QMUL(g, QMUL(bq, ak));
        row[q2 * nr + k2] = make_double2(v, 0.0);
        m = fmax(m, fabs(v));
      }
    }
  }
  if (maxabs != nullptr) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(maxabs + b, (unsigned long long)__double_as_longlong(m));
  }
}

}  // namespace qch

// ============================================================================
// host side
namespace qch {

struct Workspace {
  cudaStream_t st;
  void* p = nullptr;
  explicit Workspace(cudaStream_t s) : st(s) {}
  cudaError_t alloc(size_t bytes) {
    ensure_pool();
    return cudaMallocAsync(&p, bytes, st);
  }
  ~Workspace() {
    if (p) cudaFreeAsync(p, st);
  }
};

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

extern "C" int qch_max_abs_batch_c128(const void* d_h, int64_t batch, int64_t n_elems, double* d_out,
                                      void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (batch <= 0) return QCH_OK;
  QCH_CUDA(cudaMemsetAsync(d_out, 0, sizeof(double) * batch, st));
  if (n_elems <= 0) return QCH_OK;
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int64_t nb = std::min<int64_t>(batch - b0, 65535);
    const int per = (int)std::max<int64_t>(1, std::min<int64_t>((n_elems + 255) / 256, (int64_t)sm_count() * 8 / nb));
    max_abs_kernel<<<dim3(per, (unsigned)nb), 256, 0, st>>>((const double2*)d_h + b0 * n_elems, n_elems,
                                                            (unsigned long long*)d_out + b0);
    QCH_LAUNCH_CHECK("max_abs_kernel");
    note_launch(1);
  }
  return QCH_OK;
}

static int hermitian_tiles(const void* d_h, int64_t n, int* d_flag, double* d_defect, cudaStream_t st) {
  if (n <= 0) return QCH_OK;
  const int64_t T = (n + 31) / 32;
  const int64_t pairs = T * (T + 1) / 2;
  if (pairs > INT32_MAX) return fail(QCH_ERR_UNSUPPORTED, "hermiticity check: matrix too large");
  hermitian_tiles_kernel<<<(unsigned)pairs, 256, 0, st>>>((const double2*)d_h, n, d_flag,
                                                          (unsigned long long*)d_defect);
  QCH_LAUNCH_CHECK("hermitian_tiles_kernel");
  note_launch(1);
  return QCH_OK;
}

extern "C" int qch_hermitian_exact_c128(const void* d_h, int64_t n, int* d_nonherm, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  QCH_CUDA(cudaMemsetAsync(d_nonherm, 0, sizeof(int), st));
  return hermitian_tiles(d_h, n, d_nonherm, nullptr, st);
}

extern "C" int qch_hermitian_defect_c128(const void* d_h, int64_t n, double* d_defect, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  QCH_CUDA(cudaMemsetAsync(d_defect, 0, sizeof(double), st));
  return hermitian_tiles(d_h, n, nullptr, d_defect, st);
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
                                                 const double* d_params, double* d_maxabs, void* stream) {
  if (batch <= 0) return QCH_OK;
  if (n_q < 1 || n_r < 1) return fail(QCH_ERR_VALUE, "need n_q, n_r >= 1");
  if (n_q * n_r >= 65536) return fail(QCH_ERR_UNSUPPORTED, "builder: dimension must be < 65536");
  cudaStream_t st = (cudaStream_t)stream;
  const int n = (int)(n_q * n_r);
  if (d_maxabs) QCH_CUDA(cudaMemsetAsync(d_maxabs, 0, sizeof(double) * batch, st));
  const int bx = (int)std::max<int64_t>(1, std::min<int64_t>(n, (int64_t)sm_count() * 16 / batch + 1));
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int64_t nb = std::min<int64_t>(batch - b0, 65535);
    build_tr_kernel<<<dim3(bx, (unsigned)nb), 256, 0, st>>>((double2*)d_h + b0 * (int64_t)n * n, (int)n_q, (int)n_r,
                                                           d_params + 4 * b0,
                                                           (unsigned long long*)(d_maxabs ? d_maxabs + b0 : nullptr));
    QCH_LAUNCH_CHECK("build_tr_kernel");
    note_launch(1);
  }
  return QCH_OK;
}


// ----------------------------------------------------------------------------
// npad_run drivers (C-ABI)
#include "npad_run.h"

namespace {
using namespace qch;

struct RunBufs {
  unsigned char* mask = nullptr;
  double* q = nullptr;
  int* c = nullptr;
  double2* v = nullptr;
  NpadJob2* jobs = nullptr;
  int* flag = nullptr;
};

size_t run_bytes(int64_t batch, int n) {
  return 4096 + (size_t)n + (sizeof(double) + sizeof(int) + sizeof(double2)) * (size_t)n * batch +
         sizeof(NpadJob2) * batch;
}

RunBufs carve_run(void* base, int64_t batch, int n) {
  unsigned char* p = (unsigned char*)base;
  auto take = [&](size_t b) {
    unsigned char* q = p;
    p += (b + 255) & ~size_t(255);
    return q;
  };
  RunBufs r;
  r.flag = (int*)take(sizeof(int) * 4);
  r.jobs = (NpadJob2*)take(sizeof(NpadJob2) * batch);
  r.v = (double2*)take(sizeof(double2) * n * batch);
  r.q = (double*)take(sizeof(double) * n * batch);
  r.c = (int*)take(sizeof(int) * n * batch);
  r.mask = take(n);
  return r;
}

// exact keys when |z|^2 could leave the normal range for entries that matter
int exact_keys(double max_abs, double threshold) {
  return (max_abs > 1e100 || (threshold > 0.0 && threshold < 1e-140)) ? 1 : 0;
}

int fill_mask(unsigned char* mask, int n, const int32_t* d_target, int64_t n_target, cudaStream_t st) {
  fill_mask_kernel<<<(n + 255) / 256, 256, 0, st>>>(mask, n, d_target, (int)n_target);
  if (n_target > 0) set_mask_kernel<<<(int)((n_target + 255) / 256), 256, 0, st>>>(mask, d_target, (int)n_target);
  QCH_LAUNCH_CHECK("mask kernels");
  note_launch(n_target > 0 ? 2 : 1);
  return QCH_OK;
}
}  // namespace

extern "C" int qch_unitarity_defect_c128(const void* d_u, int64_t batch, int64_t n, double* d_defect, void* stream);

extern "C" int qch_npad_run_dense_c128(void* d_h, int64_t n, const int32_t* d_target, int64_t n_target,
                                       double threshold, int64_t max_iter, void* d_u, int32_t* d_pivots,
                                       int64_t pivot_cap, int64_t* applied, int* converged, void* stream) {
  if (n < 1) return fail(QCH_ERR_VALUE, "dimension must be at least 1");
  if (n >= 65536) return fail(QCH_ERR_UNSUPPORTED, "npad: dimension must be < 65536");
  cudaStream_t st = (cudaStream_t)stream;
  const int ni = (int)n;
  Workspace ws(st);
  QCH_CUDA(ws.alloc(run_bytes(1, ni)));
  RunBufs rb = carve_run(ws.p, 1, ni);
  if (int rc = qch_hermitian_exact_c128(d_h, n, rb.flag, stream)) return rc;
  QCH_CUDA(cudaMemsetAsync(rb.flag + 1, 0, sizeof(double), st));
  if (int rc = qch_max_abs_c128(d_h, n * n, (double*)(rb.flag + 2), stream)) return rc;
  int host[4] = {0, 0, 0, 0};
  QCH_CUDA(cudaMemcpyAsync(host, rb.flag, sizeof(host), cudaMemcpyDeviceToHost, st));
  QCH_CUDA(cudaStreamSynchronize(st));
  double maxabs;
  memcpy(&maxabs, host + 2, sizeof(double));
  const bool herm = host[0] == 0;

  NpadCommon2 cm;
  cm.n = ni;
  cm.inT = d_target ? rb.mask : nullptr;
  cm.tlist = d_target;
  cm.n_target = (int)n_target;
  cm.ek = exact_keys(maxabs, threshold);
  cm.max_iter = max_iter;
  cm.stats = getenv("QCH_NPAD_STATS") ? 1 : 0;
  const bool trows = npad_use_trows(cm, herm) && d_u == nullptr;
  if (d_target) {
    if (int rc = fill_mask(rb.mask, ni, d_target, n_target, st)) return rc;
  }
  if (int rc = npad_state_init((const double2*)d_h, 1, cm, trows, rb.q, rb.c, rb.v, st)) return rc;

  const int64_t audit_every = 100;  // UNITARY_CHECK_EVERY, npad.py:216
  // one large full-diagonal chain: the whole GPU (cooperative, npad_coop.cu).
  // With U tracking the chain pauses at every multiple of 100 rotations for
  // the audit (npad.py:254-259) and resumes from a fresh row state.
  {
    const char* e = getenv("QCH_NPAD_COOP");
    const bool coop = e ? atoi(e) != 0 : n >= 1024;
    if (coop && !trows && herm && d_target == nullptr) {
      Workspace wsd(st);
      double* d_def = nullptr;
      if (d_u) {
        QCH_CUDA(wsd.alloc(sizeof(double)));
        d_def = (double*)wsd.p;
      }
      long long total = 0;
      int stt = 0;
      bool ran = false;
      while (true) {
        long long limit = max_iter - total;
        if (d_u) limit = std::min<long long>(limit, ((total / audit_every) + 1) * audit_every - total);
        if (total > 0)
          if (int rc = npad_state_init((const double2*)d_h, 1, cm, trows, rb.q, rb.c, rb.v, st)) return rc;
        long long ap = 0;
        const int rc = npad_run_coop((double2*)d_h, ni, threshold, limit, cm.ek, rb.q, rb.c, rb.v,
                                     d_pivots ? d_pivots + 2 * std::min<long long>(total, pivot_cap) : nullptr,
                                     d_pivots ? std::max<long long>(0, pivot_cap - total) : 0, &ap, &stt, st,
                                     (double2*)d_u);
        if (rc == QCH_ERR_UNSUPPORTED && !ran) break;  // the single-CTA driver below
        if (rc != QCH_OK) return rc;
        ran = true;
        total += ap;
        if (d_u && ap > 0 && total % audit_every == 0) {
          if (int rc2 = qch_unitarity_defect_c128(d_u, 1, n, d_def, stream)) return rc2;
          double defect = 0.0;
          QCH_CUDA(cudaMemcpyAsync(&defect, d_def, sizeof(double), cudaMemcpyDeviceToHost, st));
          QCH_CUDA(cudaStreamSynchronize(st));
          if (!(defect <= 1e-10 * (double)n)) {
            char buf[160];
            snprintf(buf, sizeof buf, "accumulated unitary drift %.3e after %lld rotations", defect, total);
            return fail(QCH_ERR_UNITARITY_DRIFT, buf);
          }
        }
        if (stt == 0 || total >= max_iter) break;
      }
      if (ran) {
        *applied = total;
        *converged = stt == 0 ? 1 : 0;
        return QCH_OK;
      }
    }
  }

  NpadJob2 job;
  job.h = (double2*)d_h;
  job.u = (double2*)d_u;
  job.st_q = rb.q;
  job.st_c = rb.c;
  job.st_v = rb.v;
  job.pivots = d_pivots;
  job.pivot_cap = d_pivots ? pivot_cap : 0;
  job.threshold = threshold;
  job.applied = 0;
  job.status = 3;  // not started
  job.stats[0] = job.stats[1] = job.stats[2] = job.stats[3] = 0;
  Workspace ws2(st);
  double* d_defect = nullptr;
  if (d_u) {
    QCH_CUDA(ws2.alloc(sizeof(double)));
    d_defect = (double*)ws2.p;
  }
  while (true) {
    cm.stop_at = d_u ? ((job.applied / audit_every) + 1) * audit_every : INT64_MAX;
    QCH_CUDA(cudaMemcpyAsync(rb.jobs, &job, sizeof(NpadJob2), cudaMemcpyHostToDevice, st));
    if (int rc = npad_launch2(rb.jobs, 1, cm, herm, trows, 512, true, st)) return rc;
    QCH_CUDA(cudaMemcpyAsync(&job, rb.jobs, sizeof(NpadJob2), cudaMemcpyDeviceToHost, st));
    QCH_CUDA(cudaStreamSynchronize(st));
    if (job.status != 2) break;
    // paused at a multiple of 100 rotations: ||U U^dag - I||_F <= 1e-10 N
    if (int rc = qch_unitarity_defect_c128(d_u, 1, n, d_defect, stream)) return rc;
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

__global__ void batch_jobs_kernel(NpadJob2* jobs, double2* h, int64_t n, const double* thr, double* q, int* c,
                                  double2* v, int64_t per, int64_t batch) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= batch) return;
  NpadJob2 j;
  j.h = h + b * n * n;
  j.u = nullptr;
  j.st_q = q + b * per;
  j.st_c = c + b * per;
  j.st_v = v + b * per;
  j.pivots = nullptr;
  j.pivot_cap = 0;
  j.threshold = thr[b];
  j.applied = 0;
  j.status = 3;  // not started
  j.stats[0] = j.stats[1] = j.stats[2] = j.stats[3] = 0;
  jobs[b] = j;
}
__global__ void batch_out_kernel(const NpadJob2* jobs, int64_t batch, int64_t* applied, int32_t* conv) {
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
  QCH_CUDA(ws.alloc(run_bytes(batch, ni)));
  RunBufs rb = carve_run(ws.p, batch, ni);
  NpadCommon2 cm;
  cm.n = ni;
  cm.inT = d_target ? rb.mask : nullptr;
  cm.tlist = d_target;
  cm.n_target = (int)n_target;
  cm.ek = 0;  // builder-scale operators: |z|^2 keys are safe (see exact_keys)
  cm.max_iter = max_iter;
  cm.stop_at = INT64_MAX;
  cm.stats = getenv("QCH_NPAD_STATS") ? 1 : 0;
  const bool trows = npad_use_trows(cm, true);
  if (d_target) {
    if (int rc = fill_mask(rb.mask, ni, d_target, n_target, st)) return rc;
  }
  if (int rc = npad_state_init((const double2*)d_h, batch, cm, trows, rb.q, rb.c, rb.v, st)) return rc;
  const int64_t per = trows ? cm.n_target : ni;
  batch_jobs_kernel<<<(int)((batch + 127) / 128), 128, 0, st>>>(rb.jobs, (double2*)d_h, n, d_thresholds, rb.q, rb.c,
                                                                   rb.v, per, batch);
  note_launch(1);
  // Sweeps: the chains run concurrently on the many-chain driver (one warp
  // each) until at most one per SM is left; the survivors — the long chains
  // that set the makespan — finish on the shared-memory T-rows driver (one
  // CTA per chain, one global round trip per rotation).  A batch that fits
  // one CTA per SM starts there.  QCH_NPAD_DRIVER forces one driver;
  // QCH_NPAD_HANDOVER=k sets the hand-over point (0: never).
  const char* drv = getenv("QCH_NPAD_DRIVER");
  const size_t tsb = trows ? npad_tsmem_bytes(cm) : 0;
  int handover = sm_count();
  if (const char* e = getenv("QCH_NPAD_HANDOVER")) handover = atoi(e);
  if (drv != nullptr && strcmp(drv, "tsmem") == 0) {
    if (int rc = npad_launch_tsmem(rb.jobs, (int)batch, cm, st)) return rc;
  } else if (drv == nullptr && tsb > 0 && handover > 0 && batch <= handover) {
    if (int rc = npad_launch_tsmem(rb.jobs, (int)batch, cm, st)) return rc;
  } else if (drv == nullptr && tsb > 0 && handover > 0) {
    Workspace live(st);
    QCH_CUDA(live.alloc(sizeof(int)));
    const int nb = (int)batch;
    QCH_CUDA(cudaMemcpyAsync(live.p, &nb, sizeof(int), cudaMemcpyHostToDevice, st));
    NpadCommon2 c1 = cm;
    c1.live = (int*)live.p;
    c1.handover = handover;
    if (int rc = npad_launch_trows_warp(rb.jobs, (int)batch, c1, st)) return rc;
    if (int rc = npad_launch_tsmem(rb.jobs, (int)batch, cm, st)) return rc;
    QCH_CUDA(cudaStreamSynchronize(st));  // (the counter's memory is released at scope exit)
  } else {
    if (int rc = npad_launch2(rb.jobs, (int)batch, cm, true, trows, 256, false, st)) return rc;
  }
  batch_out_kernel<<<(int)((batch + 127) / 128), 128, 0, st>>>(rb.jobs, batch, d_applied, d_converged);
  QCH_LAUNCH_CHECK("batch_out_kernel");
  note_launch(1);
  return QCH_OK;
}
