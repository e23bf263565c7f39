// peaks.cu — FP64 roofline denominators measured on the box (MEASURED_PEAKS.json
// carries only HBM and bf16): DFMA pipe throughput and DMMA (mma.sync f64)
// tensor-pipe throughput.  Timed by the caller with CUDA events.
#include "qch_internal.h"

namespace qch {

__global__ void __launch_bounds__(256) dfma_peak_kernel(double* out, int iters, double seed) {
  double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
         a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 = fma(a0, m, c);
      a1 = fma(a1, m, c);
      a2 = fma(a2, m, c);
      a3 = fma(a3, m, c);
      a4 = fma(a4, m, c);
      a5 = fma(a5, m, c);
      a6 = fma(a6, m, c);
      a7 = fma(a7, m, c);
    }
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[0] = s;  // keep the chain alive
}

__global__ void __launch_bounds__(256) dmma_peak_kernel(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = seed - threadIdx.x * 1e-3;
  double c[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[q][0]), "+d"(c[q][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
  if (s == 12345.678) out[0] = s;
}

}  // namespace qch

using namespace qch;

// kind 0: DFMA (flops = 2 * 64 * iters * threads), kind 1: DMMA m8n8k4 (512 flops each,
// 8 per iteration per warp).  Returns the flop count of the launch in *flops.
extern "C" int qch_peak_kernel(int kind, int blocks, int iters, double* d_sink, double* flops, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (kind == 0) {
    dfma_peak_kernel<<<blocks, 256, 0, st>>>(d_sink, iters, 1.0);
    *flops = 2.0 * 64.0 * iters * 256.0 * blocks;
  } else {
    dmma_peak_kernel<<<blocks, 256, 0, st>>>(d_sink, iters, 1.0);
    *flops = 512.0 * 8.0 * iters * (256.0 / 32.0) * blocks;
  }
  QCH_LAUNCH_CHECK("peak kernel");
  note_launch(1);
  return QCH_OK;
}
