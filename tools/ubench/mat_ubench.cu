// Microbenchmark: latency of the 3x3 complex building blocks of the fused
// Magnus kernel (dependent matmul chain, dependent L2 load + matmul chain,
// shuffle-tree round), one warp alone and with the GPU full.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2411_09982_b200/csrc mat_ubench.cu
#include <cstdio>
#include "magnus_small.cuh"
using namespace qch;

__device__ __forceinline__ Mat<3> shfl_down3(const Mat<3>& m, int d) {
  Mat<3> o;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      o.v[r][c] = mkc(__shfl_down_sync(0xffffffffu, m.v[r][c].re, d), __shfl_down_sync(0xffffffffu, m.v[r][c].im, d));
  return o;
}

__global__ void k_chain(const double2* src, double2* out, int iters, int mode, long long* cyc) {
  Mat<3> m, x;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      m.v[r][c] = d2c(src[r * 3 + c]);
      x.v[r][c] = d2c(src[9 + r * 3 + c]);
    }
  const int lane = threadIdx.x & 31;
  __syncwarp();
  long long c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
    if (mode == 0) {
      m = mat_mul_fma<3>(m, x);
    } else if (mode == 1) {
      const double2* p = src + 32 + ((i * 97 + blockIdx.x * 13) & 4095) * 9;
      Mat<3> y;
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) y.v[r][c] = d2c(__ldcg(p + r * 3 + c));
      m = mat_mul_fma<3>(m, y);
    } else if (mode == 2) {
      const Mat<3> o = shfl_down3(m, 1 << (i % 5));
      if ((lane & 1) == 0) m = mat_mul_fma<3>(m, o);
    } else {
      const double2* p = src + 32 + ((i * 97 + blockIdx.x * 13) & 4095) * 9;
      Mat<3> y;
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) y.v[r][c] = d2c(__ldcg(p + r * 3 + c));
      m.v[0][0].re += y.v[0][0].re;  // load latency only
      m.v[1][1].re += y.v[2][2].im;
    }
  }
  long long c1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
  double s = 0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) s += m.v[r][c].re + m.v[r][c].im;
  if (s == 12345.0) out[0] = make_double2(s, 0);
}

int main() {
  double2* src;
  double2* out;
  long long* cyc;
  const size_t n = 32 + 4096 * 9 + 64;
  cudaMalloc(&src, n * sizeof(double2));
  cudaMalloc(&out, 16);
  cudaMalloc(&cyc, 4096 * sizeof(long long));
  double2* h = new double2[n];
  for (size_t i = 0; i < n; ++i) h[i] = make_double2(1e-3 * (i % 7), 1e-3 * (i % 5));
  cudaMemcpy(src, h, n * sizeof(double2), cudaMemcpyHostToDevice);
  const char* names[] = {"matmul chain", "ldcg+matmul chain", "shfl-tree round", "ldcg chain"};
  struct Cfg { int grid, block; } cfgs[] = {{1, 32}, {148, 128}, {444, 128}, {1184, 128}};
  for (int mode = 0; mode < 4; ++mode)
    for (auto cf : cfgs) {
      const int iters = 200;
      k_chain<<<cf.grid, cf.block>>>(src, out, iters, mode, cyc);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k_chain<<<cf.grid, cf.block>>>(src, out, iters, mode, cyc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      long long hc[4096];
      cudaMemcpy(hc, cyc, cf.grid * sizeof(long long), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int b = 0; b < cf.grid; ++b) avg += hc[b];
      avg /= cf.grid;
      printf("%-20s grid %5d x %3d: %8.1f cycles/iter (kernel %.1f us)\n", names[mode], cf.grid, cf.block, avg / iters,
             ms * 1e3);
    }
  return 0;
}
