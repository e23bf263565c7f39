// Copy-engine H2D of the config-2 signals (2 x 400001 doubles, pinned) in
// chunks: plain 1D copies per control row vs 2D copies, with and without a
// cuStreamWriteValue32 after each chunk.  Reports wall time per transfer.
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>

int main() {
  const long S = 400001, K = 2;
  double *h, *d;
  int* flag;
  cudaHostAlloc(&h, K * S * 8, cudaHostAllocMapped);
  cudaMalloc(&d, K * S * 8);
  cudaMalloc(&flag, 256);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (long i = 0; i < K * S; ++i) h[i] = i;
  auto run = [&](int nch, int mode, bool wv) {
    auto t0 = std::chrono::steady_clock::now();
    const int reps = 20;
    for (int r = 0; r < reps; ++r) {
      const long per = (S + nch - 1) / nch;
      for (int c = 0; c < nch; ++c) {
        const long s0 = c * per, s1 = (s0 + per < S) ? s0 + per : S;
        if (mode == 0) {
          cudaMemcpy2DAsync(d + s0, S * 8, h + s0, S * 8, (s1 - s0) * 8, K, cudaMemcpyHostToDevice, st);
        } else {
          for (int k = 0; k < K; ++k)
            cudaMemcpyAsync(d + k * S + s0, h + k * S + s0, (s1 - s0) * 8, cudaMemcpyHostToDevice, st);
        }
        if (wv) cuStreamWriteValue32(st, (CUdeviceptr)flag, c + 1, 0);
      }
      cudaStreamSynchronize(st);
    }
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / reps;
    printf("chunks %3d %s %-9s %8.1f us  (%.1f GB/s)\n", nch, mode == 0 ? "2D" : "1D", wv ? "+wv32" : "", us,
           K * S * 8 / us * 1e-3);
  };
  cuInit(0);
  run(1, 0, false);
  for (int nch : {1, 4, 8, 16, 32})
    for (int mode : {0, 1})
      for (bool wv : {false, true}) run(nch, mode, wv);
  return 0;
}
