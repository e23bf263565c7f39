// rk4.cu — the fixed-step RK4 comparator (reference.py:11-65) on the GPU
// (the baseline of bench_magnus / run_spin_chain).
//
// psi' = -i H(t) psi with H(t) = H0 + sum_k u_k(t) H_k read off grid samples
// (steps must satisfy 2*steps | S-1: the half-step Hamiltonian is an exact
// sample).  One launch runs all steps: G CTAs own contiguous row blocks,
// every stage is a fused SpMV over the UNION sparsity pattern of H0 and the
// H_k (each stored entry carries its K+1 operator values, so H(t) is never
// materialised), a thread per row for short rows (spin chains: 2L+1 entries)
// or a warp per row, and the four stages of a step are separated
// by grid barriers (monotone arrival counter, release/acquire; G = 1 for
// small problems: plain block barriers).  Stage s reads its input vector as
// psi + a_s k_{s-1} on the fly; the final combination writes the next
// trajectory row.  Arithmetic: complex FMAs in the order of a CSR row (the
// reference's scipy SpMV sums the same products; results agree to rounding).
#include <algorithm>
#include <cstdint>

#include "qch_internal.h"
#include "qch_math.cuh"

namespace qch {
namespace {

constexpr int kRkThreads = 256;

struct RkArgs {
  const int64_t* indptr;  // (N+1)
  const int* indices;     // (nnz)
  const double2* vals;    // (nnz, K+1): H0 value then H_1..H_K
  int n, K;
  const double* sig;      // (K, S)
  int64_t S;
  int64_t steps, stride;
  double h;
  double2* traj;          // (steps+1, N); row 0 = psi0 (set by the host)
  double2* kbuf;          // (4, N) stage derivatives
  unsigned* bar;          // grid-barrier counter (zeroed)
};

__device__ __forceinline__ void grid_sync(const RkArgs& a, unsigned& epoch) {
  __syncthreads();
  if (gridDim.x == 1) return;
  ++epoch;
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    atomicAdd(a.bar, 1u);
    const unsigned target = epoch * gridDim.x;
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

template <bool TPR>  // true: thread per row (short rows); false: warp per row
__global__ void __launch_bounds__(kRkThreads) rk4_kernel(const RkArgs a) {
  extern __shared__ double s_u[];  // (3, K): u at the step's lo / mid / hi samples
  const int n = a.n, K = a.K;
  const int G = gridDim.x;
  const int R = (n + G - 1) / G;
  const int r0 = blockIdx.x * R, r1 = min(n, r0 + R);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kRkThreads / 32;
  unsigned epoch = 0;
  const double h = a.h;
  // stage s: input x = psi + c_s k_{s-1}, coefficients at sample point p_s
  const double cin[4] = {0.0, 0.5 * h, 0.5 * h, h};
  const int pnt[4] = {0, 1, 1, 2};
  for (int64_t step = 0; step < a.steps; ++step) {
    const double2* psi = a.traj + step * n;
    if (threadIdx.x < 3 * K) {
      const int q = threadIdx.x / K, k = threadIdx.x % K;
      const int64_t idx = step * a.stride + (q == 0 ? 0 : q == 1 ? a.stride / 2 : a.stride);
      s_u[q * K + k] = a.sig[(int64_t)k * a.S + idx];
    }
    __syncthreads();
#pragma unroll 1
    for (int s = 0; s < 4; ++s) {
      const double c = cin[s];
      const double* u = s_u + pnt[s] * K;
      const double2* kprev = a.kbuf + (int64_t)(s > 0 ? s - 1 : 0) * n;
      double2* kout = a.kbuf + (int64_t)s * n;
      const int rstart = TPR ? r0 + (int)threadIdx.x : r0 + warp;
      const int rstep = TPR ? kRkThreads : nw;
      const int estart = TPR ? 0 : lane, estep = TPR ? 1 : 32;
      for (int r = rstart; r < r1; r += rstep) {
        double yr = 0.0, yi = 0.0;
        for (int64_t e = a.indptr[r] + estart; e < a.indptr[r + 1]; e += estep) {
          const int col = __ldg(a.indices + e);
          const double2* v = a.vals + e * (K + 1);
          double hr = v[0].x, hi = v[0].y;
          for (int k = 0; k < K; ++k) {
            hr = fma(u[k], v[k + 1].x, hr);
            hi = fma(u[k], v[k + 1].y, hi);
          }
          double2 x = __ldcg(psi + col);
          if (s > 0) {
            const double2 kp = __ldcg(kprev + col);
            x.x = fma(c, kp.x, x.x);
            x.y = fma(c, kp.y, x.y);
          }
          yr = fma(hr, x.x, fma(-hi, x.y, yr));
          yi = fma(hr, x.y, fma(hi, x.x, yi));
        }
        if (!TPR) {
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            yr += __shfl_xor_sync(0xffffffffu, yr, off);
            yi += __shfl_xor_sync(0xffffffffu, yi, off);
          }
        }
        if (TPR || lane == 0) __stcg(kout + r, make_double2(yi, -yr));  // k = -i H x
      }
      grid_sync(a, epoch);
    }
    // psi_{n+1} = psi + h/6 (k1 + 2 k2 + 2 k3 + k4) for this CTA's rows
    double2* nxt = a.traj + (step + 1) * n;
    const double h6 = h / 6.0;
    for (int r = r0 + threadIdx.x; r < r1; r += kRkThreads) {
      const double2 p = __ldcg(psi + r);
      const double2 k1 = __ldcg(a.kbuf + r), k2 = __ldcg(a.kbuf + n + r), k3 = __ldcg(a.kbuf + 2 * n + r),
                    k4 = __ldcg(a.kbuf + 3 * n + r);
      const double sr = k1.x + 2.0 * k2.x + 2.0 * k3.x + k4.x;
      const double si = k1.y + 2.0 * k2.y + 2.0 * k3.y + k4.y;
      __stcg(nxt + r, make_double2(p.x + h6 * sr, p.y + h6 * si));
    }
    grid_sync(a, epoch);
  }
}

}  // namespace
}  // namespace qch

using namespace qch;

extern "C" int qch_rk4_evolve_c128(const int64_t* d_indptr, const int* d_indices, const void* d_vals, int64_t n,
                                   int64_t K, const double* d_sig, int64_t S, double t_start, double t_end,
                                   int64_t steps, const void* d_psi0, void* d_traj, void* stream) {
  if (n < 1) return fail(QCH_ERR_VALUE, "dimension must be at least 1");
  if (steps < 1) return fail(QCH_ERR_GRID, "need at least one step");
  if ((S - 1) % (2 * steps))
    return fail(QCH_ERR_GRID, std::to_string(steps) + " RK steps need 2*steps to divide " + std::to_string(S - 1) +
                                  " sample steps");
  if (K > 32) return fail(QCH_ERR_UNSUPPORTED, "at most 32 control channels");
  cudaStream_t st = (cudaStream_t)stream;
  RkArgs a;
  a.indptr = d_indptr;
  a.indices = d_indices;
  a.vals = (const double2*)d_vals;
  a.n = (int)n;
  a.K = (int)K;
  a.sig = d_sig;
  a.S = S;
  a.steps = steps;
  a.stride = (S - 1) / steps;
  a.h = (t_end - t_start) / (double)steps;
  a.traj = (double2*)d_traj;
  void* ws = nullptr;
  ensure_pool();
  QCH_CUDA(cudaMallocAsync(&ws, sizeof(double2) * 4 * (size_t)n + 256, st));
  a.kbuf = (double2*)((unsigned char*)ws + 256);
  a.bar = (unsigned*)ws;
  QCH_CUDA(cudaMemsetAsync(ws, 0, 256, st));
  QCH_CUDA(cudaMemcpyAsync(d_traj, d_psi0, sizeof(double2) * n, cudaMemcpyDeviceToDevice, st));
  // nnz from the row pointer (one 8-byte read)
  int64_t nnz = 0;
  QCH_CUDA(cudaMemcpyAsync(&nnz, d_indptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  QCH_CUDA(cudaStreamSynchronize(st));
  // short rows (< 32 entries on average): a thread per row, one CTA per 256
  // rows; long rows: a warp per row, one CTA per ~16k entries; at most one
  // CTA per SM (grid barriers), one CTA needs only block barriers
  const bool tpr = nnz < 32 * n;
  const int64_t want = tpr ? (n + kRkThreads - 1) / kRkThreads : nnz / 16384;
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>(sm_count(), want));
  const size_t smem = sizeof(double) * 3 * std::max<int64_t>(K, 1);
  auto kern = tpr ? rk4_kernel<true> : rk4_kernel<false>;
  void* pr = prof_begin("rk4_kernel", st);
  if (G > 1) {
    void* args[] = {(void*)&a};
    QCH_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(G), dim3(kRkThreads), args, smem, st));
  } else {
    kern<<<1, kRkThreads, smem, st>>>(a);
  }
  prof_end(pr, st);
  QCH_LAUNCH_CHECK("rk4_kernel");
  note_launch(1);
  QCH_CUDA(cudaFreeAsync(ws, st));
  QCH_CUDA(cudaStreamSynchronize(st));
  return QCH_OK;
}
