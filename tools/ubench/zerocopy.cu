// Zero-copy host-link throughput from SMs (mapped pinned memory): reads of
// 16 KB windows into shared memory (cp.async 8 B / 16 B, cp.async.bulk) with
// one or two windows in flight per block, and 16 B stores of a trajectory.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

constexpr int kThreads = 128;
constexpr int kWin = 16384;  // bytes per window

__device__ __forceinline__ void cpa8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cpa16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int W>
__device__ __forceinline__ void waitg() { asm volatile("cp.async.wait_group %0;\n" ::"n"(W) : "memory"); }

__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk(void* s, const void* g, unsigned bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(s)),
               "l"(g), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(b))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(b)),
      "r"(phase)
      : "memory");
}

__global__ void rd(const char* src, long nwin, int mode, int depth, double* sink) {
  extern __shared__ __align__(128) char sm[];
  __shared__ uint64_t bar[2];
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double acc = 0;
  unsigned ph[2] = {0, 0};
  auto issue = [&](long w, int buf) {
    char* dst = sm + buf * kWin;
    const char* s = src + w * kWin;
    if (mode == 0) {
      for (int q = threadIdx.x; q < kWin / 8; q += kThreads) cpa8(dst + q * 8, s + q * 8);
      commit();
    } else if (mode == 1) {
      for (int q = threadIdx.x; q < kWin / 16; q += kThreads) cpa16(dst + q * 16, s + q * 16);
      commit();
    } else if (threadIdx.x == 0) {
      mbar_expect(&bar[buf], kWin);
      bulk(dst, s, kWin, &bar[buf]);
    }
  };
  int it = 0;
  long w = blockIdx.x;
  if (w < nwin) issue(w, 0);
  for (; w < nwin; w += gridDim.x, ++it) {
    const int buf = it & 1;
    const long wn = w + gridDim.x;
    if (depth == 2 && wn < nwin) issue(wn, buf ^ 1);
    if (mode < 2) {
      if (depth == 2 && wn < nwin) waitg<1>(); else waitg<0>();
    } else {
      mbar_wait(&bar[buf], ph[buf]);
      ph[buf] ^= 1;
    }
    __syncthreads();
    acc += ((double*)(sm + buf * kWin))[threadIdx.x];
    __syncthreads();
    if (depth == 1 && wn < nwin) issue(wn, buf ^ 1);
  }
  if (acc == 1234.5) sink[0] = acc;
}

__global__ void wr(double2* dst, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    dst[i] = make_double2(i, -i);
}

int main() {
  const long bytes = 6400000 / kWin * kWin;
  char* h;
  cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  for (long i = 0; i < bytes; ++i) h[i] = (char)i;
  char* d;
  cudaHostGetDevicePointer(&d, h, 0);
  double* sink;
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(rd, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kWin);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"cp.async 8B", "cp.async 16B", "cp.async.bulk"};
  for (int grid : {148, 296})
    for (int mode = 0; mode < 3; ++mode)
      for (int depth = 1; depth <= 2; ++depth) {
        rd<<<grid, kThreads, 2 * kWin>>>(d, bytes / kWin, mode, depth, sink);
        cudaEventRecord(e0);
        for (int r = 0; r < 10; ++r) rd<<<grid, kThreads, 2 * kWin>>>(d, bytes / kWin, mode, depth, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("read  grid %3d %-14s depth %d: %7.1f us  %.1f GB/s  (%s)\n", grid, names[mode], depth, ms * 100,
               bytes / (ms * 1e-4) * 1e-9, cudaGetErrorString(cudaGetLastError()));
      }
  const long n = 4800000 / 16;
  double2* ht;
  cudaHostAlloc(&ht, n * 16, cudaHostAllocMapped);
  double2* dt;
  cudaHostGetDevicePointer(&dt, ht, 0);
  for (int grid : {148, 296, 1184}) {
    wr<<<grid, 128>>>(dt, n);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) wr<<<grid, 128>>>(dt, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("write grid %4d 16B stores: %7.1f us  %.1f GB/s\n", grid, ms * 100, n * 16 / (ms * 1e-4) * 1e-9);
  }
  return 0;
}
