// builders.cu — device-side model builders: the
// controlled spin chain of the experiment runners (models.py:288-325) built
// as device CSR operators, so a chain sweep never builds or uploads on the
// host.  Bit-identical to the host builders (same integer sums, the same
// rounded products and differences, scipy's CSR layout: sorted columns,
// explicit zeros of the diagonal dropped).
#include <cstdint>

#include "qch_internal.h"
#include "qch_math.cuh"

namespace qch {
namespace {

constexpr int kBThreads = 1024;

// z_j = 1 - 2 bit_j; diagonal = (0.5 w) sum z - J sum z_j z_{j+1} - g2 sum z_j z_{j+2}
// (periodic), evaluated as numpy does: ((0.5*w)*S1 - J*S2) - g2*S3.
__device__ __forceinline__ double chain_diag(int64_t b, int L, double hw, double jn, double g2) {
  int s1 = 0, s2 = 0, s3 = 0;
  for (int j = 0; j < L; ++j) {
    const int zj = 1 - 2 * (int)((b >> j) & 1);
    const int z1 = 1 - 2 * (int)((b >> ((j + 1) % L)) & 1);
    const int z2 = 1 - 2 * (int)((b >> ((j + 2) % L)) & 1);
    s1 += zj;
    s2 += zj * z1;
    s3 += zj * z2;
  }
  return QSUB(QSUB(QMUL(hw, (double)s1), QMUL(jn, (double)s2)), QMUL(g2, (double)s3));
}

// one CTA: each thread owns a contiguous run of rows; nonzero diagonal
// entries are compacted with a block scan (scipy drops explicit zeros)
__global__ void __launch_bounds__(kBThreads) chain_drift_kernel(int L, double hw, double jn, double g2,
                                                                int64_t* __restrict__ indptr,
                                                                int32_t* __restrict__ indices,
                                                                double2* __restrict__ data, int64_t* __restrict__ nnz) {
  const int64_t n = (int64_t)1 << L;
  const int64_t per = (n + kBThreads - 1) / kBThreads;
  const int64_t r0 = threadIdx.x * per, r1 = min(n, r0 + per);
  int cnt = 0;
  for (int64_t r = r0; r < r1; ++r) cnt += chain_diag(r, L, hw, jn, g2) != 0.0 ? 1 : 0;
  // exclusive block scan of the counts
  __shared__ int s_w[kBThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) s_w[w] = x;
  __syncthreads();
  if (w == 0) {
    int v = lane < kBThreads / 32 ? s_w[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, v, d);
      if (lane >= d) v += y;
    }
    if (lane < kBThreads / 32) s_w[lane] = v;  // inclusive warp totals
  }
  __syncthreads();
  int64_t off = (int64_t)(x - cnt) + (w > 0 ? s_w[w - 1] : 0);
  for (int64_t r = r0; r < r1; ++r) {
    indptr[r] = off;
    const double d = chain_diag(r, L, hw, jn, g2);
    if (d != 0.0) {
      indices[off] = (int32_t)r;
      data[off] = make_double2(d, 0.0);
      ++off;
    }
  }
  if (threadIdx.x == kBThreads - 1) {
    indptr[n] = off;
    *nnz = off;
  }
}

// sum_j sx_j and sum_j sy_j: row r holds columns r ^ (1 << j), sorted; sy's
// entry (r, r ^ 2^j) is +i when bit j of r is set (the source state has it
// clear), -i otherwise (models.py:313-320)
__global__ void global_xy_kernel(int L, int64_t* __restrict__ ipx, int32_t* __restrict__ ixx,
                                 double2* __restrict__ dvx, int64_t* __restrict__ ipy, int32_t* __restrict__ ixy,
                                 double2* __restrict__ dvy) {
  const int64_t n = (int64_t)1 << L;
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r > n) return;
  ipx[r] = r * L;
  ipy[r] = r * L;
  if (r == n) return;
  int64_t cols[32];
  for (int j = 0; j < L; ++j) cols[j] = r ^ ((int64_t)1 << j);
  for (int a = 1; a < L; ++a) {  // insertion sort (L <= 30)
    const int64_t v = cols[a];
    int b = a - 1;
    while (b >= 0 && cols[b] > v) {
      cols[b + 1] = cols[b];
      --b;
    }
    cols[b + 1] = v;
  }
  for (int j = 0; j < L; ++j) {
    const int64_t c = cols[j];
    const int site = __ffsll((long long)(c ^ r)) - 1;
    const bool set = (r >> site) & 1;
    ixx[r * L + j] = (int32_t)c;
    dvx[r * L + j] = make_double2(1.0, 0.0);
    ixy[r * L + j] = (int32_t)c;
    dvy[r * L + j] = make_double2(0.0, set ? 1.0 : -1.0);
  }
}

}  // namespace
}  // namespace qch

using namespace qch;

extern "C" int qch_build_spin_chain_drift_c128(int64_t length, double qubit_freq, double j_nn, double g_nnn,
                                               int64_t* d_indptr, int32_t* d_indices, void* d_data, int64_t* nnz,
                                               void* stream) {
  if (length < 1 || length > 30) return fail(QCH_ERR_VALUE, "spin chain length must be within [1, 30]");
  cudaStream_t st = (cudaStream_t)stream;
  int64_t* d_nnz = nullptr;
  ensure_pool();
  QCH_CUDA(cudaMallocAsync(&d_nnz, sizeof(int64_t), st));
  chain_drift_kernel<<<1, kBThreads, 0, st>>>((int)length, QMUL(0.5, qubit_freq), j_nn, g_nnn, d_indptr, d_indices,
                                             (double2*)d_data, d_nnz);
  QCH_LAUNCH_CHECK("chain_drift_kernel");
  note_launch(1);
  QCH_CUDA(cudaMemcpyAsync(nnz, d_nnz, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  QCH_CUDA(cudaFreeAsync(d_nnz, st));
  QCH_CUDA(cudaStreamSynchronize(st));
  return QCH_OK;
}

extern "C" int qch_build_global_xy_c128(int64_t length, int64_t* d_indptr_x, int32_t* d_indices_x, void* d_data_x,
                                        int64_t* d_indptr_y, int32_t* d_indices_y, void* d_data_y, void* stream) {
  if (length < 1 || length > 30) return fail(QCH_ERR_VALUE, "spin chain length must be within [1, 30]");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = (int64_t)1 << length;
  global_xy_kernel<<<(unsigned)((n + 256) / 256), 256, 0, st>>>((int)length, d_indptr_x, d_indices_x,
                                                                  (double2*)d_data_x, d_indptr_y, d_indices_y,
                                                                  (double2*)d_data_y);
  QCH_LAUNCH_CHECK("global_xy_kernel");
  note_launch(1);
  return QCH_OK;
}
