// Cluster exchange latency: barrier.cluster (arrive.release + wait.acquire)
// vs. an all-to-all of remote mbarrier arrivals (each CTA arrives on every
// CTA's barrier, waits on its own), G = 16 CTAs in one non-portable cluster.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cs cluster_sync.cu && /tmp/cs
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void bar_kernel(int iters, long long* out) {
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cg::this_cluster().sync();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
}

__global__ void mbar_kernel(int iters, long long* out) {
  __shared__ __align__(8) unsigned long long bar[2];
  const unsigned G = cg::this_cluster().num_blocks();
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar[b])), "r"(G));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cg::this_cluster().sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const int b = i & 1;
    const unsigned local = (unsigned)__cvta_generic_to_shared(&bar[b]);
    if (threadIdx.x < G) {  // lane d arrives on CTA d's barrier
      unsigned remote;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"((unsigned)threadIdx.x));
      asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
    }
    if (threadIdx.x == 0) {
      asm volatile(
          "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(local),
          "r"((unsigned)((i >> 1) & 1))
          : "memory");
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
  cg::this_cluster().sync();
}

int main() {
  long long* d;
  cudaMalloc(&d, 64 * sizeof(long long));
  for (int G : {2, 4, 8, 16}) {
    for (int which = 0; which < 2; ++which) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(G);
      cfg.blockDim = dim3(256);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = G;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      if (which == 0) {
        cudaFuncSetAttribute(bar_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchKernelEx(&cfg, bar_kernel, 20000, d);
      } else {
        cudaFuncSetAttribute(mbar_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchKernelEx(&cfg, mbar_kernel, 20000, d);
      }
      cudaError_t e = cudaDeviceSynchronize();
      long long h[64];
      cudaMemcpy(h, d, G * sizeof(long long), cudaMemcpyDeviceToHost);
      printf("G=%2d %-22s %s cycles/round (CTA0) %lld\n", G, which ? "mbarrier all-to-all" : "barrier.cluster",
             e ? cudaGetErrorString(e) : "ok", h[0]);
    }
  }
  return 0;
}
