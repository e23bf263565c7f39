// i8gemm.cu — tcgen05 (5th-gen tensor core) int8 GEMM with TMEM accumulators:
// C_i32 (M x N) = A_i8 (M x K, K-contiguous) . B_i8 (N x K, K-contiguous)^T.
// The building block of the FP64-exact-sliced (Ozaki) complex GEMM.
//
// Warp roles (192 threads): warp 0 = TMA producer (one lane), warp 1 = TMEM
// allocator + MMA issuer (one lane), warps 2-5 = epilogue (TMEM -> registers
// -> global).  Tiles 128 x 128, K stage 128 bytes (one 128-byte swizzle row),
// 4 UMMA k-steps of 32 per stage, 6-stage smem ring with full/empty
// mbarriers; the MMA commits each stage back to its empty barrier and the
// accumulator to a TMEM-full barrier.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "qch_internal.h"

namespace qch {

constexpr int I8_BM = 128, I8_BK = 128;
constexpr int I8_THREADS = 192;

__device__ __forceinline__ unsigned i8_smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void i8_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n I8_W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra I8_W;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void i8_tma2(unsigned dst, const CUtensorMap* map, int c0, int c1, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

// K-major, 128-byte swizzle smem matrix descriptor (UMMA::SmemDescriptor):
// start >> 4 [0,14), LBO >> 4 [16,30) (unused for swizzled K-major), SBO >> 4
// [32,46) = 1024 B between 8-row groups, version 1 [46,48), layout 2 (128B
// swizzle) [61,64)
__device__ __forceinline__ uint64_t i8_desc(unsigned saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// instruction descriptor kind::i8: D s32 [4,6)=2, A s8 [7,10)=1, B s8
// [10,13)=1, K-major A/B, N >> 3 at [17,23), M >> 4 at [24,29)
constexpr uint32_t i8_idesc(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

template <int I8_BN>
__global__ void __launch_bounds__(I8_THREADS, 1)
    i8gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int32_t* c, int m,
                  int n, int k) {
  constexpr int I8_ST = I8_BN == 128 ? 6 : 4;
  constexpr int I8_STAGE = (I8_BM + I8_BN) * I8_BK;
  extern __shared__ unsigned char i8_raw[];
  unsigned char* base = (unsigned char*)(((uintptr_t)i8_raw + 1023) & ~(uintptr_t)1023);
  unsigned long long* full = (unsigned long long*)(base + I8_ST * I8_STAGE);
  unsigned long long* empty = full + I8_ST;
  unsigned long long* accf = empty + I8_ST;  // accumulator ready
  unsigned* s_tmem = (unsigned*)(accf + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tn = (n + I8_BN - 1) / I8_BN;
  const int ti = blockIdx.x / tn, tj = blockIdx.x % tn;
  const int m0 = ti * I8_BM, n0 = tj * I8_BN;
  const int KT = (k + I8_BK - 1) / I8_BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < I8_ST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(i8_smem_u32(full + s)) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(i8_smem_u32(empty + s)) : "memory");
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(i8_smem_u32(accf)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // TMEM: 128 lanes x 128 columns of s32
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(i8_smem_u32(s_tmem)),
                 "n"(I8_BN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = *s_tmem;

  if (warp == 0) {
    if (lane == 0) {
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % I8_ST;
        i8_wait(i8_smem_u32(empty + s), (unsigned)(((kt / I8_ST) & 1) ^ 1));
        const unsigned fb = i8_smem_u32(full + s);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(I8_STAGE) : "memory");
        const unsigned dA = i8_smem_u32(base + s * I8_STAGE);
        i8_tma2(dA, &tmA, kt * I8_BK, m0, fb);
        i8_tma2(dA + I8_BM * I8_BK, &tmB, kt * I8_BK, n0, fb);
        if (I8_BN == 256) i8_tma2(dA + (I8_BM + 128) * I8_BK, &tmB, kt * I8_BK, n0 + 128, fb);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = i8_idesc(I8_BM, I8_BN);
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % I8_ST;
        i8_wait(i8_smem_u32(full + s), (unsigned)((kt / I8_ST) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const unsigned a0 = i8_smem_u32(base + s * I8_STAGE);
        const unsigned b0 = a0 + I8_BM * I8_BK;
#pragma unroll
        for (int kk = 0; kk < I8_BK / 32; ++kk) {
          const uint64_t da = i8_desc(a0 + kk * 32), db = i8_desc(b0 + kk * 32);
          const unsigned acc = (kt > 0 || kk > 0) ? 1u : 0u;
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
              "l"(da), "l"(db), "r"(idesc), "r"(acc)
              : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         i8_smem_u32(empty + s))
                     : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       i8_smem_u32(accf))
                   : "memory");
    }
  } else {  // epilogue warps 2..5: TMEM lane quarter (warp % 4)
    i8_wait(i8_smem_u32(accf), 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int q = warp & 3;
    const int row = m0 + q * 32 + lane;
#pragma unroll 1
    for (int cb = 0; cb < I8_BN; cb += 32) {
      uint32_t v[32];
      const unsigned taddr = tmem + ((unsigned)(q * 32) << 16) + (unsigned)cb;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
          "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
            "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
            "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
            "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (row < m)
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (n0 + cb + e < n) c[(int64_t)row * n + n0 + cb + e] = (int32_t)v[e];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(I8_BN) : "memory");
}

static PFN_cuTensorMapEncodeTiled_v12000 i8_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

static int i8_map(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int box_rows) {
  box_rows = std::min(box_rows, 128);
  auto fn = i8_encode();
  if (!fn) return fail(QCH_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols};
  cuuint32_t box[2] = {(cuuint32_t)I8_BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)ptr, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(QCH_ERR_CUDA, "cuTensorMapEncodeTiled (i8) failed (" + std::to_string((int)r) + ")");
  return QCH_OK;
}

}  // namespace qch

using namespace qch;

// experimental: C (M x N int32) = A (M x K int8) . B (N x K int8)^T; K % 16 == 0
template <int BN>
static int i8_run(const void* d_a, const void* d_b, void* d_c, int64_t m, int64_t n, int64_t k, cudaStream_t st) {
  CUtensorMap ma, mb;
  if (int rc = i8_map(&ma, d_a, m, k, I8_BM)) return rc;
  if (int rc = i8_map(&mb, d_b, n, k, 128)) return rc;
  constexpr int ST = BN == 128 ? 6 : 4;
  const int smem = ST * (I8_BM + BN) * I8_BK + 1024 + 256;
  QCH_CUDA(smem_attr((const void*)i8gemm_kernel<BN>, smem));
  const int tiles = (int)(((m + I8_BM - 1) / I8_BM) * ((n + BN - 1) / BN));
  void* pr = prof_begin("i8gemm", st);
  i8gemm_kernel<BN><<<tiles, I8_THREADS, smem, st>>>(ma, mb, (int32_t*)d_c, (int)m, (int)n, (int)k);
  prof_end(pr, st);
  QCH_LAUNCH_CHECK("i8gemm_kernel");
  note_launch(1);
  return QCH_OK;
}

// experimental: C (M x N int32) = A (M x K int8) . B (N x K int8)^T; K % 16 == 0; bn 128 | 256
extern "C" int qch_i8gemm_test(const void* d_a, const void* d_b, void* d_c, int64_t m, int64_t n, int64_t k,
                               void* stream) {
  if (k % 16) return fail(QCH_ERR_VALUE, "i8gemm: K must be a multiple of 16");
  static const int bn = getenv("QCH_I8_BN") ? atoi(getenv("QCH_I8_BN")) : 128;
  if (bn == 256) return i8_run<256>(d_a, d_b, d_c, m, n, k, (cudaStream_t)stream);
  return i8_run<128>(d_a, d_b, d_c, m, n, k, (cudaStream_t)stream);
}
