// GPU-side duration of an empty kernel vs parameter size and dynamic shared
// memory (CUDA events around each launch, back to back).
#include <cuda_runtime.h>
#include <cstdio>

struct Big { double v[340]; };  // ~2.7 KB, like FusedArgs
__global__ void k_small(int x) { if (x == 12345) printf("x"); }
__global__ void k_big(const __grid_constant__ Big b) { if (b.v[0] == 12345.0) printf("x"); }
__global__ void k_smem(int x) {
  extern __shared__ double s[];
  if (x == 12345) s[threadIdx.x] = 1;
}

int main() {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  Big b = {};
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 72 * 1024);
  for (int rep = 0; rep < 2; ++rep) {
    for (int mode = 0; mode < 4; ++mode) {
      float tot = 0;
      for (int i = 0; i < 50; ++i) {
        cudaEventRecord(e0);
        if (mode == 0) k_small<<<391, 128>>>(1);
        if (mode == 1) k_big<<<391, 128>>>(b);
        if (mode == 2) k_smem<<<391, 128, 70528>>>(1);
        if (mode == 3) k_small<<<1, 32>>>(1);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        tot += ms;
      }
      const char* nm[] = {"small params, 391x128", "2.7 KB params, 391x128", "70 KB smem, 391x128", "1x32"};
      printf("%-26s %.2f us\n", nm[mode], tot / 50 * 1e3);
    }
  }
  return 0;
}
