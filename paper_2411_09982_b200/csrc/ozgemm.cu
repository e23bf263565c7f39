// ozgemm.cu — FP64-accurate real GEMMs on the int8 tensor cores (tcgen05
// kind::i8, TMEM accumulators) by exact slicing (the Ozaki scheme), and the
// Hermitian complex products of exp(-iH) built from them.
//
// Slicing.  Row r of a real operand X is scaled by 2^-e_r (e_r: the frexp
// exponent of the row's max |x|, so |x 2^-e_r| < 1) and cut into s int8
// slices, 7 bits each: t = 128 x; a = trunc(t) (|a| <= 127); x = t - a — all
// exact in FP64.  X[r,k] = 2^e_r sum_i a_i[r,k] 2^-7(i+1) + O(2^(e_r - 7s)).
// Product.  (X Y^T)[r,c] = 2^(e_r + f_c) sum_{i,j} 2^-7(i+j+2) (a_i b_j^T)[r,c];
// the int8 products are EXACT in int32 (K 127^2 (i+j+1) < 2^31 for K <= 4096,
// s <= 8) and the pairs with i + j <= s - 1 are kept (s(s+1)/2 int8 GEMMs):
// the dropped tail and the slicing residual are below 2^-7s relative to
// 2^(e_r + f_c) K — s = 7 gives ~1e-15 of the row/column scale, the FP64
// rounding level of a K = 4096 dot product.  One kernel per real product:
// for each diagonal D = i + j the pairs accumulate in one TMEM buffer (int32),
// the epilogue warps fold it into FP64 registers as 2^-7(D+2) D_int, the two
// TMEM buffers alternating so the MMAs of diagonal D+1 overlap the epilogue of
// diagonal D.
//
// Warp roles (320 threads): warp 0 TMA producer (one lane), warp 1 TMEM
// allocator + MMA issuer (one lane), warps 2-9 epilogue (warp w: TMEM lane
// quarter w % 4, columns 64 ((w-2) / 4) ..).  Tile 128 x 128, K stage 128 B
// (one 128-byte swizzle row), 4 UMMA k-steps (K = 32) per stage, 6 stages.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <vector>

#include "qch_internal.h"

namespace qch {

constexpr int OZ_BM = 128, OZ_BN = 128, OZ_BK = 128, OZ_ST = 6;
constexpr int OZ_STAGE = (OZ_BM + OZ_BN) * OZ_BK;  // 32 KB
constexpr int OZ_EPI_WARPS = 8;
constexpr int OZ_THREADS = (2 + OZ_EPI_WARPS) * 32;
constexpr int OZ_MAX_S = 8;

__device__ __forceinline__ unsigned oz_smem(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void oz_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n OZ_W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra OZ_W;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void oz_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void oz_tma3(unsigned dst, const CUtensorMap* map, int c0, int c1, int c2, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

// K-major, 128-byte-swizzle UMMA smem descriptor (SBO = 1024 B per 8 rows)
__device__ __forceinline__ uint64_t oz_desc(unsigned saddr) {
  return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
// kind::i8 instruction descriptor: D s32, A/B signed int8, K-major, M, N
constexpr uint32_t oz_idesc(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

struct OzArgs {
  const int* ea;   // [batch][m] row exponents of X
  const int* eb;   // [batch][n] row exponents of Y
  double* out;     // [batch][m][ldo] (P = X Y^T)
  int m, n, k, s;  // s slices
  int ldo;
  int64_t so;      // batch stride of out
  const int* tiles;  // optional tile list (ti << 16 | tj); null: all tiles
  int ntiles;        // tiles per batch item
  int tn;
};

__global__ void __launch_bounds__(OZ_THREADS, 1)
    oz_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, OzArgs g) {
  extern __shared__ unsigned char oz_raw[];
  unsigned char* base = (unsigned char*)(((uintptr_t)oz_raw + 1023) & ~(uintptr_t)1023);
  unsigned long long* full = (unsigned long long*)(base + OZ_ST * OZ_STAGE);
  unsigned long long* empty = full + OZ_ST;
  unsigned long long* tfull = empty + OZ_ST;  // [2] accumulator buffer ready
  unsigned long long* tempty = tfull + 2;     // [2] accumulator buffer drained
  unsigned* s_tmem = (unsigned*)(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bz = blockIdx.y;
  int ti, tj;
  if (g.tiles) {
    const int t = g.tiles[blockIdx.x];
    ti = t >> 16;
    tj = t & 0xffff;
  } else {
    ti = blockIdx.x / g.tn;
    tj = blockIdx.x % g.tn;
  }
  const int m0 = ti * OZ_BM, n0 = tj * OZ_BN;
  const int KT = (g.k + OZ_BK - 1) / OZ_BK;
  const int S = g.s;

  if (threadIdx.x == 0) {
    for (int q = 0; q < OZ_ST; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(oz_smem(full + q)) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(oz_smem(empty + q)) : "memory");
    }
    for (int q = 0; q < 2; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(oz_smem(tfull + q)) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(oz_smem(tempty + q)), "r"(OZ_EPI_WARPS)
                   : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // TMEM: 128 lanes x 256 columns = two 128-column int32 accumulators
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(oz_smem(s_tmem))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = *s_tmem;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer: (D, i, kt) in the MMA issuer's order
      int it = 0;
      for (int D = 0; D < S; ++D)
        for (int i = 0; i <= D; ++i)
          for (int kt = 0; kt < KT; ++kt, ++it) {
            const int q = it % OZ_ST;
            oz_wait(oz_smem(empty + q), (unsigned)(((it / OZ_ST) & 1) ^ 1));
            const unsigned fb = oz_smem(full + q);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(OZ_STAGE) : "memory");
            const unsigned dA = oz_smem(base + q * OZ_STAGE);
            oz_tma3(dA, &tmA, kt * OZ_BK, m0, bz * S + i, fb);
            oz_tma3(dA + OZ_BM * OZ_BK, &tmB, kt * OZ_BK, n0, bz * S + (D - i), fb);
          }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = oz_idesc(OZ_BM, OZ_BN);
      int it = 0;
      for (int D = 0; D < S; ++D) {
        const int buf = D & 1;
        oz_wait(oz_smem(tempty + buf), (unsigned)(((D >> 1) & 1) ^ 1));  // drained by the epilogue
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const unsigned tacc = tmem + (unsigned)(buf * OZ_BN);
        for (int i = 0; i <= D; ++i)
          for (int kt = 0; kt < KT; ++kt, ++it) {
            const int q = it % OZ_ST;
            oz_wait(oz_smem(full + q), (unsigned)((it / OZ_ST) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const unsigned a0 = oz_smem(base + q * OZ_STAGE);
            const unsigned b0 = a0 + OZ_BM * OZ_BK;
#pragma unroll
            for (int kk = 0; kk < OZ_BK / 32; ++kk) {
              const uint64_t da = oz_desc(a0 + kk * 32), db = oz_desc(b0 + kk * 32);
              const unsigned acc = (i > 0 || kt > 0 || kk > 0) ? 1u : 0u;
              asm volatile(
                  "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                  " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tacc),
                  "l"(da), "l"(db), "r"(idesc), "r"(acc)
                  : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             oz_smem(empty + q))
                         : "memory");
          }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         oz_smem(tfull + buf))
                     : "memory");
      }
    }
  } else {  // epilogue: FP64 accumulation of the diagonals
    const int q4 = warp & 3, half = (warp - 2) >> 2;
    const int row = m0 + q4 * 32 + lane;
    double acc[64];
#pragma unroll
    for (int e = 0; e < 64; ++e) acc[e] = 0.0;
    for (int D = 0; D < S; ++D) {
      const int buf = D & 1;
      oz_wait(oz_smem(tfull + buf), (unsigned)((D >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const double scl = ldexp(1.0, -7 * (D + 2));
#pragma unroll
      for (int cb = 0; cb < 64; cb += 32) {
        uint32_t v[32];
        const unsigned taddr = tmem + ((unsigned)(q4 * 32) << 16) + (unsigned)(buf * OZ_BN + half * 64 + cb);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
            "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int e = 0; e < 32; ++e) acc[cb + e] = fma((double)(int)v[e], scl, acc[cb + e]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) oz_arrive(oz_smem(tempty + buf));
    }
    if (row < g.m) {
      const int er = g.ea[(int64_t)bz * g.m + row];
      double* orow = g.out + (int64_t)bz * g.so + (int64_t)row * g.ldo;
      const int* ebb = g.eb + (int64_t)bz * g.n;
#pragma unroll
      for (int e = 0; e < 64; ++e) {
        const int c = n0 + half * 64 + e;
        if (c < g.n) orow[c] = ldexp(acc[e], er + ebb[c]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

// Slices of one real component of a batch of complex matrices, row by row:
// comp 0: Re, 1: Im, 2: Re + Im, 3: Re - Im, 4: -Im.  One block per (item, row).
__global__ void __launch_bounds__(256) oz_slice_kernel(const double2* __restrict__ x, int rows, int cols,
                                                       int64_t xstride, int comp, int s, int8_t* __restrict__ sl,
                                                       int* __restrict__ ex) {
  const int r = blockIdx.x;
  const int64_t b = blockIdx.y;
  const double2* xr = x + b * xstride + (int64_t)r * cols;
  auto val = [&](double2 v) {
    switch (comp) {
      case 0: return v.x;
      case 1: return v.y;
      case 2: return v.x + v.y;
      case 3: return v.x - v.y;
      default: return -v.y;
    }
  };
  double m = 0.0;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) m = fmax(m, fabs(val(xr[c])));
  __shared__ double s_m[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = m;
  __syncthreads();
  m = s_m[0];
  for (int w = 1; w < 8; ++w) m = fmax(m, s_m[w]);
  int e = 0;
  if (m > 0.0) frexp(m, &e);  // m = f 2^e, f in [0.5, 1): |x 2^-e| < 1
  if (threadIdx.x == 0) ex[b * rows + r] = e;
  const int64_t plane = (int64_t)rows * cols;
  int8_t* out = sl + b * (int64_t)s * plane + (int64_t)r * cols;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    double t = ldexp(val(xr[c]), -e);
    for (int i = 0; i < s; ++i) {
      t *= 128.0;
      const double a = trunc(t);
      t -= a;
      out[(int64_t)i * plane + c] = (int8_t)(int)a;
    }
  }
}

// The three components of one operand role in ONE pass over the complex
// matrix (it is read once instead of three times): comps c0, c1, c2 as
// oz_slice_kernel, slice sets sl0/sl1/sl2, exponents ex0/ex1/ex2.
__device__ __forceinline__ double oz_comp(double2 v, int comp) {
  switch (comp) {
    case 0: return v.x;
    case 1: return v.y;
    case 2: return v.x + v.y;
    case 3: return v.x - v.y;
    default: return -v.y;
  }
}

__global__ void __launch_bounds__(256) oz_slice3_kernel(const double2* __restrict__ x, int rows, int cols,
                                                        int64_t xstride, int c0, int c1, int c2, int s,
                                                        int8_t* __restrict__ sl0, int8_t* __restrict__ sl1,
                                                        int8_t* __restrict__ sl2, int* __restrict__ ex0,
                                                        int* __restrict__ ex1, int* __restrict__ ex2) {
  const int r = blockIdx.x;
  const int64_t b = blockIdx.y;
  const double2* xr = x + b * xstride + (int64_t)r * cols;
  double m0 = 0.0, m1 = 0.0, m2 = 0.0;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    const double2 v = xr[c];
    m0 = fmax(m0, fabs(oz_comp(v, c0)));
    m1 = fmax(m1, fabs(oz_comp(v, c1)));
    m2 = fmax(m2, fabs(oz_comp(v, c2)));
  }
  __shared__ double s_m[3][8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    m0 = fmax(m0, __shfl_xor_sync(0xffffffffu, m0, o));
    m1 = fmax(m1, __shfl_xor_sync(0xffffffffu, m1, o));
    m2 = fmax(m2, __shfl_xor_sync(0xffffffffu, m2, o));
  }
  if ((threadIdx.x & 31) == 0) {
    s_m[0][threadIdx.x >> 5] = m0;
    s_m[1][threadIdx.x >> 5] = m1;
    s_m[2][threadIdx.x >> 5] = m2;
  }
  __syncthreads();
  int e[3];
  for (int q = 0; q < 3; ++q) {
    double m = s_m[q][0];
    for (int w = 1; w < 8; ++w) m = fmax(m, s_m[q][w]);
    e[q] = 0;
    if (m > 0.0) frexp(m, &e[q]);
  }
  if (threadIdx.x == 0) {
    ex0[b * rows + r] = e[0];
    ex1[b * rows + r] = e[1];
    ex2[b * rows + r] = e[2];
  }
  const int64_t plane = (int64_t)rows * cols;
  const int64_t off = b * (int64_t)s * plane + (int64_t)r * cols;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    const double2 v = xr[c];
    double t0 = ldexp(oz_comp(v, c0), -e[0]), t1 = ldexp(oz_comp(v, c1), -e[1]), t2 = ldexp(oz_comp(v, c2), -e[2]);
    for (int i = 0; i < s; ++i) {
      t0 *= 128.0;
      t1 *= 128.0;
      t2 *= 128.0;
      const double a0 = trunc(t0), a1 = trunc(t1), a2 = trunc(t2);
      t0 -= a0;
      t1 -= a1;
      t2 -= a2;
      const int64_t o = off + (int64_t)i * plane + c;
      sl0[o] = (int8_t)(int)a0;
      sl1[o] = (int8_t)(int)a1;
      sl2[o] = (int8_t)(int)a2;
    }
  }
}

static int oz_slice3(const double2* x, int n, int64_t batch, const int* comps, int s, int8_t* const* sl,
                     int* const* ex, cudaStream_t st) {
  const int64_t nn = (int64_t)n * n;
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int64_t nb = std::min<int64_t>(batch - b0, 65535);
    const int64_t so = b0 * (int64_t)s * nn;
    void* pr = prof_begin("oz_slice", st);
    oz_slice3_kernel<<<dim3(n, (unsigned)nb), 256, 0, st>>>(x + b0 * nn, n, n, nn, comps[0], comps[1], comps[2], s,
                                                             sl[0] + so, sl[1] + so, sl[2] + so, ex[0] + b0 * n,
                                                             ex[1] + b0 * n, ex[2] + b0 * n);
    prof_end(pr, st);
    QCH_LAUNCH_CHECK("oz_slice3_kernel");
    note_launch(1);
  }
  return QCH_OK;
}

static PFN_cuTensorMapEncodeTiled_v12000 oz_encode() {
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

// slices [planes][rows][cols] int8 as a 3-d map, box 128 B x 128 rows
static int oz_map(CUtensorMap* map, const int8_t* ptr, int64_t rows, int64_t cols, int64_t planes) {
  auto fn = oz_encode();
  if (!fn) return fail(QCH_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)cols, (cuuint64_t)(rows * cols)};
  cuuint32_t box[3] = {(cuuint32_t)OZ_BK, 128u, 1u};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)ptr, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(QCH_ERR_CUDA, "cuTensorMapEncodeTiled (oz) failed (" + std::to_string((int)r) + ")");
  return QCH_OK;
}

int oz_slice(const double2* x, int rows, int cols, int64_t batch, int64_t xstride, int comp, int s, int8_t* sl, int* ex,
             cudaStream_t st) {
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int64_t nb = std::min<int64_t>(batch - b0, 65535);
    void* pr = prof_begin("oz_slice", st);
    oz_slice_kernel<<<dim3(rows, (unsigned)nb), 256, 0, st>>>(x + b0 * xstride, rows, cols, xstride, comp, s,
                                                               sl + b0 * (int64_t)s * rows * cols, ex + b0 * rows);
    prof_end(pr, st);
    QCH_LAUNCH_CHECK("oz_slice_kernel");
    note_launch(1);
  }
  return QCH_OK;
}

// P_b = X_b Y_b^T for a batch (slices as produced by oz_slice); tiles: null =
// all tiles, else a device list of ntiles (ti << 16 | tj)
int oz_gemm(const int8_t* xs, const int* ea, const int8_t* ys, const int* eb, int m, int n, int k, int s,
            int64_t batch, double* out, int ldo, int64_t so, const int* tiles, int ntiles, cudaStream_t st) {
  if (s < 1 || s > OZ_MAX_S) return fail(QCH_ERR_VALUE, "ozaki: 1..8 slices");
  // exact int32 accumulation: (slices per diagonal) K 127^2 < 2^31
  if (k % 16 || (int64_t)s * k * 127 * 127 >= (int64_t)1 << 31)
    return fail(QCH_ERR_UNSUPPORTED, "ozaki: K must be a multiple of 16 and s K 127^2 < 2^31");
  CUtensorMap ma, mb;
  if (int rc = oz_map(&ma, xs, m, k, batch * s)) return rc;
  if (int rc = oz_map(&mb, ys, n, k, batch * s)) return rc;
  const int smem = OZ_ST * OZ_STAGE + 1024 + 256;
  static bool attr = false;
  if (!attr) {
    QCH_CUDA(cudaFuncSetAttribute(oz_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  OzArgs g{};
  g.ea = ea;
  g.eb = eb;
  g.out = out;
  g.m = m;
  g.n = n;
  g.k = k;
  g.s = s;
  g.ldo = ldo;
  g.so = so;
  g.tiles = tiles;
  g.tn = (n + OZ_BN - 1) / OZ_BN;
  g.ntiles = tiles ? ntiles : ((m + OZ_BM - 1) / OZ_BM) * g.tn;
  void* pr = prof_begin("oz_gemm", st);
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int64_t nb = std::min<int64_t>(batch - b0, 65535);
    (void)nb;
    if (b0 > 0) return fail(QCH_ERR_UNSUPPORTED, "ozaki: batch > 65535");
    oz_gemm_kernel<<<dim3(g.ntiles, (unsigned)batch), OZ_THREADS, smem, st>>>(ma, mb, g);
    QCH_LAUNCH_CHECK("oz_gemm_kernel");
    note_launch(1);
  }
  prof_end(pr, st);
  return QCH_OK;
}

// C = A B for batches of Hermitian n x n A, B whose product is Hermitian
// (commuting Hermitian polynomials of one matrix), by the Gauss / 3M form on
// three Ozaki real products over the tiles meeting the lower triangle:
//   P1 = Ar Br,  P2 = Ai Bi,  P3 = (Ar + Ai)(Br + Bi)
//   Re = P1 - P2,  Im = P3 - P1 - P2
// The Y operands are rows of B^T = conj(B): Br, -Bi, Br - Bi.  The combine
// pass applies the epilogue (STORE / QACC / UFIN as zgemm_tma.cu) on r >= c
// and writes the conjugate mirror.
struct OzCombine {
  const double* p1;
  const double* p2;
  const double* p3;
  double2* c;
  const double2* pw[4];  // QACC: P_1..P_nq ; UFIN: pw[0] = C (cos part)
  double q[5];
  int nq;
  int mode;  // 0 STORE, 2 QACC, 3 UFIN (zgemm.h numbering)
  int n;
};

__global__ void oz_combine_kernel(OzCombine a, int64_t batch) {
  const int64_t nn = (int64_t)a.n * a.n;
  const int64_t total = nn * batch;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = k / nn, e = k - b * nn;
    const int r = (int)(e / a.n), c = (int)(e - (int64_t)r * a.n);
    if (r < c) continue;
    const double v1 = a.p1[k], v2 = a.p2[k], v3 = a.p3[k];
    const double re = v1 - v2, im = (v3 - v1) - v2;
    const int64_t moff = b * nn + (int64_t)c * a.n + r;
    if (a.mode == 3) {  // U = C - i S
      const double2 cv = a.pw[0][k];
      a.c[k] = make_double2(cv.x + im, cv.y - re);
      if (r > c) a.c[moff] = make_double2(cv.x - im, -cv.y - re);
      continue;
    }
    double xr = re, xi = im;
    if (a.mode == 2) {
      xr += (r == c) ? a.q[0] : 0.0;
      for (int i = 0; i < a.nq; ++i) {
        const double2 pv = a.pw[i][k];
        xr = fma(a.q[i + 1], pv.x, xr);
        xi = fma(a.q[i + 1], pv.y, xi);
      }
    }
    a.c[k] = make_double2(xr, xi);
    if (r > c) a.c[moff] = make_double2(xr, -xi);
  }
}

static int oz_lower_tiles(int n, const int** out, int* count, cudaStream_t st) {
  static int cached_n = -1, cached_cnt = 0;
  static int* d_list = nullptr;
  if (cached_n != n) {
    // lower-triangle tiles in 8 x 8 super-tiles, so the ~148 concurrent CTAs
    // share A and B slice panels (an L2-resident working set)
    const int T = (n + OZ_BM - 1) / OZ_BM;
    std::vector<int> h;
    for (int bi = 0; bi < T; bi += 8)
      for (int bj = 0; bj <= bi; bj += 8)
        for (int i = bi; i < std::min(T, bi + 8); ++i)
          for (int j = bj; j < std::min(bj + 8, i + 1); ++j) h.push_back((i << 16) | j);
    if (d_list) cudaFree(d_list);
    QCH_CUDA(cudaMalloc((void**)&d_list, sizeof(int) * h.size()));
    QCH_CUDA(cudaMemcpyAsync(d_list, h.data(), sizeof(int) * h.size(), cudaMemcpyHostToDevice, st));
    QCH_CUDA(cudaStreamSynchronize(st));
    cached_n = n;
    cached_cnt = (int)h.size();
  }
  *out = d_list;
  *count = cached_cnt;
  return QCH_OK;
}

// which engine takes the Hermitian products: 1 = int8 tensor cores (Ozaki,
// default), 0 = DMMA; QCH_HERM_GEMM=dmma or qch_set_herm_gemm(0) selects DMMA
static int g_herm_engine = -1;
int herm_engine() {
  if (g_herm_engine < 0) {
    const char* e = getenv("QCH_HERM_GEMM");
    g_herm_engine = (e && strcmp(e, "dmma") == 0) ? 0 : 1;
  }
  return g_herm_engine;
}
void set_herm_engine(int v) { g_herm_engine = v ? 1 : 0; }

int oz_slices() {
  static const int v = getenv("QCH_OZ_SLICES") ? std::max(1, std::min(OZ_MAX_S, atoi(getenv("QCH_OZ_SLICES")))) : 8;
  return v;
}

static std::atomic<double> g_i8_ops{0.0};
double oz_int8_ops_total() { return g_i8_ops.load(); }

int zgemm_herm_ozaki(int mode, const double2* a, const double2* b, double2* c, const double2* const* pw,
                     const double* q, int nq, int n, int64_t batch, cudaStream_t st) {
  const int S = oz_slices();
  const int64_t nn = (int64_t)n * n;
  const size_t sl_bytes = (size_t)S * nn * batch;  // one slice set
  const size_t ex_bytes = sizeof(int) * (size_t)n * batch;
  const size_t p_bytes = sizeof(double) * (size_t)nn * batch;
  ensure_pool();
  unsigned char* ws = nullptr;
  const size_t total = 6 * sl_bytes + 6 * ex_bytes + 3 * p_bytes + 6 * 256;
  QCH_CUDA(cudaMallocAsync((void**)&ws, total, st));
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  unsigned char* p = ws;
  int8_t* xs[3];
  int8_t* ys[3];
  int* ea[3];
  int* eb[3];
  for (int v = 0; v < 3; ++v) {
    xs[v] = (int8_t*)p;
    p += al(sl_bytes);
    ys[v] = (int8_t*)p;
    p += al(sl_bytes);
    ea[v] = (int*)p;
    p += al(ex_bytes);
    eb[v] = (int*)p;
    p += al(ex_bytes);
  }
  double* P[3];
  for (int v = 0; v < 3; ++v) {
    P[v] = (double*)p;
    p += al(p_bytes);
  }
  const int xc[3] = {0, 1, 2}, yc[3] = {0, 4, 3};
  int rc = QCH_OK;
  const int* tiles = nullptr;
  int ntiles = 0;
  rc = oz_lower_tiles(n, &tiles, &ntiles, st);
  if (rc == QCH_OK) rc = oz_slice3(a, n, batch, xc, S, xs, ea, st);
  if (rc == QCH_OK) rc = oz_slice3(b, n, batch, yc, S, ys, eb, st);
  for (int v = 0; v < 3 && rc == QCH_OK; ++v)
    rc = oz_gemm(xs[v], ea[v], ys[v], eb[v], n, n, n, S, batch, P[v], n, nn, tiles, ntiles, st);
  if (rc == QCH_OK) {
    double ops = 3.0 * ntiles * (double)OZ_BM * OZ_BN * n * 2.0 * (S * (S + 1) / 2) * batch;
    double cur = g_i8_ops.load();
    while (!g_i8_ops.compare_exchange_weak(cur, cur + ops)) {
    }
    OzCombine cm{};
    cm.p1 = P[0];
    cm.p2 = P[1];
    cm.p3 = P[2];
    cm.c = c;
    cm.nq = nq;
    cm.mode = mode;
    cm.n = n;
    for (int i = 0; i < 4; ++i) cm.pw[i] = (pw && i < (mode == 3 ? 1 : nq)) ? pw[i] : nullptr;
    for (int i = 0; i < 5; ++i) cm.q[i] = (q && i <= nq) ? q[i] : 0.0;
    const int blocks = (int)std::min<int64_t>((nn * batch + 255) / 256, (int64_t)sm_count() * 16);
    void* pr = prof_begin("oz_combine", st);
    oz_combine_kernel<<<blocks, 256, 0, st>>>(cm, batch);
    prof_end(pr, st);
    note_launch(1);
    if (cudaGetLastError() != cudaSuccess) rc = fail(QCH_ERR_CUDA, "oz_combine_kernel launch failed");
  }
  cudaFreeAsync(ws, st);
  return rc;
}

}  // namespace qch

using namespace qch;

extern "C" int qch_set_herm_gemm(int engine) {
  const int old = herm_engine();
  if (engine >= 0) set_herm_engine(engine);
  return old;
}

extern "C" double qch_int8_ops(void) { return oz_int8_ops_total(); }

// experimental: P (m x n, f64) = X Y^T for real components of complex matrices
// x (m x k) and y (n x k) (comp as oz_slice_kernel), s slices
extern "C" int qch_oz_real_test(const void* d_x, int xcomp, const void* d_y, int ycomp, void* d_out, int64_t m,
                                int64_t n, int64_t k, int s, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int8_t *xs = nullptr, *ys = nullptr;
  int *ea = nullptr, *eb = nullptr;
  ensure_pool();
  QCH_CUDA(cudaMallocAsync((void**)&xs, (size_t)s * m * k, st));
  QCH_CUDA(cudaMallocAsync((void**)&ys, (size_t)s * n * k, st));
  QCH_CUDA(cudaMallocAsync((void**)&ea, sizeof(int) * m, st));
  QCH_CUDA(cudaMallocAsync((void**)&eb, sizeof(int) * n, st));
  int rc = oz_slice((const double2*)d_x, (int)m, (int)k, 1, m * k, xcomp, s, xs, ea, st);
  if (!rc) rc = oz_slice((const double2*)d_y, (int)n, (int)k, 1, n * k, ycomp, s, ys, eb, st);
  if (!rc) rc = oz_gemm(xs, ea, ys, eb, (int)m, (int)n, (int)k, s, 1, (double*)d_out, (int)n, m * n, nullptr, 0, st);
  cudaFreeAsync(xs, st);
  cudaFreeAsync(ys, st);
  cudaFreeAsync(ea, st);
  cudaFreeAsync(eb, st);
  return rc;
}
