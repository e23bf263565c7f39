// ozgemm.cu — FP64-accurate real GEMMs on the int8 tensor cores (tcgen05
// kind::i8, TMEM accumulators) by exact slicing (the Ozaki scheme), and the
// Hermitian complex products of exp(-iH) built from them.
//
// Slicing.  Row r of a real operand X is scaled by 2^-e_r (e_r: the frexp
// exponent of the row's max |x|, so |x 2^-e_r| < 1) and cut into s int8
// slices of 7 bits — the base-128 digits of |x 2^-e_r| with the sign of x:
// X[r,k] = 2^e_r sum_i a_i[r,k] 2^-7(i+1) + O(2^(e_r - 7s)).
// Product.  (X Y^T)[r,c] = 2^(e_r + f_c) sum_{i,j} 2^-7(i+j+2) (a_i b_j^T)[r,c];
// the int8 products are EXACT in int32 (K 127^2 (i+j+1) < 2^31 for K <= 16384,
// s <= 8) and the pairs with i + j <= s - 1 are kept (s(s+1)/2 int8 GEMMs):
// the dropped tail and the slicing residual are below ~2^-7s of
// 2^(e_r + f_c) K — s = 8 is the FP64 rounding level of the dot product.
// A product may use only the leading s' < s slices of a stored cut (the
// digits of a shorter cut are the leading digits of a longer one).
//
// GEMM kernels (one launch per real product; for each diagonal D = i + j the
// pairs accumulate in one of two TMEM buffers while the epilogue warps fold
// the other into FP64):
//  * oz_gemmw_kernel<256, true> (default): a CTA pair (cta_group::2) owns a
//    256 x 256 tile; each CTA stages 128 A rows + 128 B rows per 128-byte K
//    block (TMA, 128-byte swizzle, 6 stages), the even CTA issues the M = 256
//    MMAs, the diagonals are folded into the output in global memory (store,
//    then FP64 reductions at L2 with the exponents applied per contribution);
//  * oz_gemmw_kernel<256, false> / <128, true>: one CTA 128 x 256, pair
//    256 x 128 (QCH_OZ_CFG=w256 / p128);
//  * oz_gemm_kernel: one CTA, 128 x 128, FP64 accumulators in registers
//    (QCH_OZ_CFG=r128; the first version, the baseline of the others).
// Warp roles (320 threads): warp 0 TMA producer (one lane), warp 1 TMEM
// allocator + MMA issuer (one lane), warps 2-9 epilogue (warp w: TMEM lane
// quarter w % 4, column half (w - 2) / 4).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "zgemm.h"

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
  int m, n, k, s;  // s: leading slices used (digits), <= sp
  int sp;          // slice planes stored per batch item
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
            oz_tma3(dA, &tmA, kt * OZ_BK, m0, bz * g.sp + i, fb);
            oz_tma3(dA + OZ_BM * OZ_BK, &tmB, kt * OZ_BK, n0, bz * g.sp + (D - i), fb);
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

// I 2^k exactly (I an int32 diagonal sum): one multiply by a constructed
// power of two in the normal range, ldexp outside it
__device__ __forceinline__ double oz_scaled(int I, int k) {
  const double x = (double)I;
  if (k >= -1022 && k <= 1023) return x * __longlong_as_double((long long)(k + 1023) << 52);
  return ldexp(x, k);
}

// ---- wide / CTA-pair variants: FP64 accumulation in the output ----
// The 128 x 128 kernel above keeps its FP64 accumulator in registers (64 per
// epilogue thread), which caps the tile at 128 columns: per 128 x 128 x 32
// MMA it stages 8 KB through shared memory (TMA write + MMA read = 2 x 8 KB
// per 68 clk at int8 peak, well above the 128 B/clk shared-memory port).
// Here the epilogue folds each diagonal straight into the output in global
// memory: diagonal 0 is stored, later ones are FP64 reductions at L2
// (red.global.add.f64, no read round trip), each contribution already
// carrying its full power of two D_int 2^(e_r + f_c - 7(D+2)) — exact, so the
// sums round exactly as the register version's FMAs followed by the final
// ldexp; the epilogue of diagonal D overlaps the MMAs of D+1), so the tile
// can be 128 x 256 (one CTA, TMEM 2 x 256
// columns) or 256 x BN on a CTA pair (cta_group::2: the MMA issued by the
// even CTA reads A rows 0..127 / 128..255 and B rows 0..BN/2-1 / BN/2..BN-1
// from the even / odd CTA's shared memory; each CTA's TMEM holds its own 128
// rows).  Pair barriers: both CTAs' TMA bytes land on the even CTA's full[q];
// the MMA commits multicast to both CTAs' empty[q] and tfull[b]; both CTAs'
// epilogue warps arrive on the even CTA's tempty[b].
constexpr unsigned OZ_PEER_MASK = 0xFEFFFFFFu;  // shared::cluster address -> even CTA of the pair

__device__ __forceinline__ void oz_tma3_pair(unsigned dst, const CUtensorMap* map, int c0, int c1, int c2,
                                             unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4}], [%5];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar & OZ_PEER_MASK)
      : "memory");
}
__device__ __forceinline__ void oz_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int BN, bool PAIR>
struct OzW {
  static constexpr int BROWS = PAIR ? BN / 2 : BN;           // B rows staged per CTA
  static constexpr int STAGE = (OZ_BM + BROWS) * OZ_BK;      // bytes per CTA per K block
  static constexpr int ST = (200 * 1024) / STAGE;            // pipeline depth
  static constexpr int SMEM = ST * STAGE + 1024 + 256;
  static constexpr int TCOLS = 2 * BN;                       // two accumulator buffers
};

template <int BN, bool PAIR>
__global__ void __launch_bounds__(OZ_THREADS, 1)
    oz_gemmw_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, OzArgs g) {
  using W = OzW<BN, PAIR>;
  extern __shared__ unsigned char oz_raw[];
  unsigned char* base = (unsigned char*)(((uintptr_t)oz_raw + 1023) & ~(uintptr_t)1023);
  unsigned long long* full = (unsigned long long*)(base + W::ST * W::STAGE);
  unsigned long long* empty = full + W::ST;
  unsigned long long* tfull = empty + W::ST;
  unsigned long long* tempty = tfull + 2;
  unsigned* s_tmem = (unsigned*)(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned rank = 0;
  if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int bz = blockIdx.y;
  const int tile = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  int ti, tj;  // ti: (PAIR ? 256 : 128)-row block, tj: BN-column block
  if (g.tiles) {
    const int t = g.tiles[tile];
    ti = t >> 16;
    tj = t & 0xffff;
  } else {
    ti = tile / g.tn;
    tj = tile % g.tn;
  }
  const int m0 = ti * (PAIR ? 2 : 1) * OZ_BM + (int)rank * OZ_BM;  // this CTA's A rows / output rows
  const int n0 = tj * BN;                                         // output columns
  const int nb0 = n0 + (int)rank * W::BROWS;                      // this CTA's B rows
  const int KT = (g.k + OZ_BK - 1) / OZ_BK;
  const int S = g.s;

  if (threadIdx.x == 0) {
    for (int q = 0; q < W::ST; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(oz_smem(full + q)) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(oz_smem(empty + q)) : "memory");
    }
    for (int q = 0; q < 2; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(oz_smem(tfull + q)) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(oz_smem(tempty + q)),
                   "r"((PAIR ? 2 : 1) * OZ_EPI_WARPS)
                   : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if (PAIR) {  // the same warp in both CTAs allocates the pair's TMEM
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(oz_smem(s_tmem)),
                   "n"(W::TCOLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(oz_smem(s_tmem)),
                   "n"(W::TCOLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (PAIR)
    oz_cluster_sync();  // barriers of both CTAs initialised, TMEM allocated
  else
    __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = *s_tmem;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer: own A rows + own B rows (PAIR: onto the even CTA's full[q])
      int it = 0;
      for (int D = 0; D < S; ++D)
        for (int i = 0; i <= D; ++i)
          for (int kt = 0; kt < KT; ++kt, ++it) {
            const int q = it % W::ST;
            oz_wait(oz_smem(empty + q), (unsigned)(((it / W::ST) & 1) ^ 1));
            const unsigned fb = oz_smem(full + q);
            const unsigned dA = oz_smem(base + q * W::STAGE);
            if (PAIR) {
              if (rank == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(2 * W::STAGE)
                             : "memory");
              oz_tma3_pair(dA, &tmA, kt * OZ_BK, m0, bz * g.sp + i, fb);
              oz_tma3_pair(dA + OZ_BM * OZ_BK, &tmB, kt * OZ_BK, nb0, bz * g.sp + (D - i), fb);
            } else {
              asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(W::STAGE)
                           : "memory");
              oz_tma3(dA, &tmA, kt * OZ_BK, m0, bz * g.sp + i, fb);
              oz_tma3(dA + OZ_BM * OZ_BK, &tmB, kt * OZ_BK, nb0, bz * g.sp + (D - i), fb);
            }
          }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // MMA issuer (the even CTA for a pair)
      constexpr uint32_t idesc = oz_idesc(PAIR ? 2 * OZ_BM : OZ_BM, BN);
      int it = 0;
      for (int D = 0; D < S; ++D) {
        const int buf = D & 1;
        oz_wait(oz_smem(tempty + buf), (unsigned)(((D >> 1) & 1) ^ 1));  // drained by the epilogue(s)
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const unsigned tacc = tmem + (unsigned)(buf * BN);
        for (int i = 0; i <= D; ++i)
          for (int kt = 0; kt < KT; ++kt, ++it) {
            const int q = it % W::ST;
            oz_wait(oz_smem(full + q), (unsigned)((it / W::ST) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const unsigned a0 = oz_smem(base + q * W::STAGE);
            const unsigned b0 = a0 + OZ_BM * OZ_BK;
#pragma unroll
            for (int kk = 0; kk < OZ_BK / 32; ++kk) {
              const uint64_t da = oz_desc(a0 + kk * 32), db = oz_desc(b0 + kk * 32);
              const unsigned acc = (i > 0 || kt > 0 || kk > 0) ? 1u : 0u;
              if (PAIR)
                asm volatile(
                    "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                    " tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tacc),
                    "l"(da), "l"(db), "r"(idesc), "r"(acc)
                    : "memory");
              else
                asm volatile(
                    "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                    " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tacc),
                    "l"(da), "l"(db), "r"(idesc), "r"(acc)
                    : "memory");
            }
            if (PAIR)
              asm volatile(
                  "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], "
                  "%1;" ::"r"(oz_smem(empty + q)),
                  "h"((unsigned short)3)
                  : "memory");
            else
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                               oz_smem(empty + q))
                           : "memory");
          }
        if (PAIR)
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  oz_smem(tfull + buf)),
              "h"((unsigned short)3)
              : "memory");
        else
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           oz_smem(tfull + buf))
                       : "memory");
      }
    }
  } else {  // epilogue: row (lane quarter q4) x BN/2 columns, folded into the output in global memory
    const int q4 = warp & 3, half = (warp - 2) >> 2;
    const int row = m0 + q4 * 32 + lane;
    const bool rok = row < g.m;
    double* orow = g.out + (int64_t)bz * g.so + (int64_t)(rok ? row : 0) * g.ldo;
    const int er = rok ? g.ea[(int64_t)bz * g.m + row] : 0;
    const int* ebb = g.eb + (int64_t)bz * g.n;
    unsigned tempty_even[2];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      tempty_even[b] = oz_smem(tempty + b);
      if (PAIR) asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(tempty_even[b]) : "r"(tempty_even[b]));
    }
    for (int D = 0; D < S; ++D) {
      const int buf = D & 1;
      oz_wait(oz_smem(tfull + buf), (unsigned)((D >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int kD = er - 7 * (D + 2);  // + the column exponent: the contribution's power of two
#pragma unroll 1
      for (int cb = 0; cb < BN / 2; cb += 32) {
        uint32_t v[32];
        const unsigned taddr =
            tmem + ((unsigned)(q4 * 32) << 16) + (unsigned)(buf * BN + half * (BN / 2) + cb);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
            "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int c0 = n0 + half * (BN / 2) + cb;
        if (rok && c0 < g.n) {
          double* o = orow + c0;
          if (D == 0) {  // first diagonal: plain stores (paired; ldo is even, so 16-byte aligned; a pair
                         // straddling column n writes the row's padding column)
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
              if (c0 + e >= g.n) break;
              const int e1 = c0 + e + 1 < g.n ? c0 + e + 1 : c0 + e;
              *(double2*)(o + e) = make_double2(oz_scaled((int)v[e], kD + ebb[c0 + e]),
                                                oz_scaled((int)v[e + 1], kD + ebb[e1]));
            }
          } else {  // later diagonals: fire-and-forget FP64 reductions at L2 (no read round trip)
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              if (c0 + e >= g.n) break;
              atomicAdd(o + e, oz_scaled((int)v[e], kD + ebb[c0 + e]));
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (PAIR)
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(tempty_even[buf])
                       : "memory");
        else
          oz_arrive(tempty_even[buf]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (PAIR) {
    oz_cluster_sync();  // the pair's MMAs and remote arrivals are complete
    if (warp == 1)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(W::TCOLS) : "memory");
  } else if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(W::TCOLS) : "memory");
  }
}

// Slices of up to four real components of a batch of complex matrices (comp
// 0: Re, 1: Im, 2: Re + Im, 3: Re - Im, 4: -Im), all components of a matrix
// from the same two passes: oz_rowexp_kernel (one block per (item, row): the
// row maxima -> exponents e) and oz_cut_kernel (every 8 consecutive columns
// independently, 8 bytes per slice plane).  The slices are the base-128
// digits of |x 2^-e| with the sign of x: |A| = |trunc(x 2^(7s - e))| < 2^7s is
// formed exactly from the bits of x (integer shift of the significand) and
// slice i = sign (|A| >> 7 (s - 1 - i)) & 127 — the same digits as the
// iteration t <- 128 t, a_i = trunc(t), t <- t - a_i.
__device__ __forceinline__ double oz_comp(double2 v, int comp) {
  switch (comp) {
    case 0: return v.x;
    case 1: return v.y;
    case 2: return v.x + v.y;
    case 3: return v.x - v.y;
    default: return -v.y;
  }
}

// slice row stride in bytes: columns rounded up to 16 (the TMA stride unit)
__host__ __device__ __forceinline__ int oz_ld(int cols) { return (cols + 15) & ~15; }

struct OzSliceOut {
  int8_t* sl[4];  // [batch][s][rows][cols]
  int* ex[4];     // [batch][rows]
  int comp[4];
  int nc;
};

// pass 1: the row exponents e (frexp of the row max of each component)
__global__ void __launch_bounds__(256) oz_rowexp_kernel(const double2* __restrict__ x, int rows, int cols,
                                                        int64_t xstride, OzSliceOut o) {
  // one WARP per row (8 rows per block): no block barrier, 8 row loads in
  // flight per lane
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int64_t b = blockIdx.y;
  const double2* xr = x + b * xstride + (int64_t)r * cols;
  double m[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
  for (int c = lane; c < cols; c += 32) {
    const double2 v = xr[c];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q < o.nc) m[q] = fmax(m[q], fabs(oz_comp(v, o.comp[q])));
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (q >= o.nc) break;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m[q] = fmax(m[q], __shfl_xor_sync(0xffffffffu, m[q], off));
    if (lane == q) {
      int e = 0;
      if (m[q] > 0.0) frexp(m[q], &e);  // m = f 2^e, f in [0.5, 1): |x| < 2^e
      o.ex[q][b * rows + r] = e;
    }
  }
}

// |trunc(y 2^(7S - e))| from the bits of y (exact: y = m 2^ex, |y| < 2^e)
template <int S>
__device__ __forceinline__ unsigned long long oz_fixed(double y, int e) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(y);
  const int ef = (int)((bits >> 52) & 0x7FF);
  const unsigned long long m = (bits & 0xFFFFFFFFFFFFFull) | (ef ? (1ull << 52) : 0ull);
  const int t = (ef ? ef : 1) - 1075 + 7 * S - e;
  return t >= 0 ? (m << t) : (t > -64 ? (m >> -t) : 0ull);
}

// the same |A| = floor(|y| 2^(7S - e)) as its two 28-bit halves, on the FP64
// pipe instead of 64-bit integer shifts: u = |y| 2^(7S-28-e) < 2^28 (exact:
// a power-of-two scaling), hi = floor(u) and lo = floor((u - hi) 2^28), each
// floor read from the low word of x + 2^52 added with round-toward-zero
// (exact: u - hi by Sterbenz, the products by powers of two; a result below
// the normal range only where the digit is 0 anyway).  Valid while the scale
// 2^(7S-28-e) is a normal double: 7S - 1051 <= e <= 7S + 994 (oz_cut_fp_ok).
template <int S>
__device__ __forceinline__ bool oz_cut_fp_ok(int e) {
  return e >= 7 * S - 1051 && e <= 7 * S + 994;
}
template <int S>
__device__ __forceinline__ void oz_halves(double y, int e, bool fp, unsigned& hi, unsigned& lo) {
  if (fp) {
    constexpr double k52 = 4503599627370496.0;  // 2^52
    const double u = fabs(y) * __longlong_as_double((long long)(7 * S - 28 - e + 1023) << 52);
    const double hb = __dadd_rz(u, k52);
    hi = (unsigned)__double2loint(hb);
    lo = (unsigned)__double2loint(__dadd_rz((u - (hb - k52)) * 268435456.0, k52));
  } else {
    const unsigned long long mg = oz_fixed<S>(y, e);
    hi = (unsigned)(mg >> 28);
    lo = (unsigned)mg & 0x0FFFFFFFu;
  }
}

// pass 2: every (item, row, 8 columns) independently — 8 consecutive columns
// per thread, 8 bytes per slice plane
template <int S>
__global__ void __launch_bounds__(256) oz_cut_kernel(const double2* __restrict__ x, int rows, int cols,
                                                     int64_t xstride, OzSliceOut o, int64_t groups, int fpcut) {
  const int ld = oz_ld(cols);  // slice row stride: padding columns are written as zeros
  const int gpr = ld >> 3;
  const int64_t plane = (int64_t)rows * ld;
  for (int64_t gi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gi < groups;
       gi += (int64_t)gridDim.x * blockDim.x) {
    const int64_t br = gi / gpr;  // b * rows + r
    const int c8 = (int)(gi - br * gpr) * 8;
    const int64_t b = br / rows;
    const int r = (int)(br - b * rows);
    const double2* xr = x + b * xstride + (int64_t)r * cols + c8;
    double2 v[8];
    if (c8 + 8 <= cols) {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = xr[j];
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = c8 + j < cols ? xr[j] : make_double2(0.0, 0.0);
    }
    const int64_t off = b * (int64_t)S * plane + (int64_t)r * ld + c8;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (q >= o.nc) break;
      const int e = o.ex[q][br];
      const bool fp = fpcut && oz_cut_fp_ok<S>(e);
      // |A| = hi 2^28 + lo (28-bit halves); digit i = bits [7(S-1-i), +7)
      unsigned hi[8], lo[8], nm0 = 0, nm1 = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double y = oz_comp(v[j], o.comp[q]);
        oz_halves<S>(y, e, fp, hi[j], lo[j]);
        if (y < 0.0) {
          if (j < 4) nm0 |= 0xFFu << (8 * j);
          else nm1 |= 0xFFu << (8 * (j - 4));
        }
      }
      int8_t* dst = o.sl[q] + off;
#pragma unroll
      for (int i = 0; i < S; ++i) {
        const int sh = 7 * (S - 1 - i);
        unsigned u[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) u[j] = sh >= 28 ? hi[j] >> (sh - 28) : lo[j] >> sh;
        unsigned w0 = __byte_perm(__byte_perm(u[0], u[1], 0x0040), __byte_perm(u[2], u[3], 0x0040), 0x5410);
        unsigned w1 = __byte_perm(__byte_perm(u[4], u[5], 0x0040), __byte_perm(u[6], u[7], 0x0040), 0x5410);
        w0 = __vsub4((w0 & 0x7F7F7F7Fu) ^ nm0, nm0);  // per-byte sign: -d = (d ^ 0xFF) - 0xFF
        w1 = __vsub4((w1 & 0x7F7F7F7Fu) ^ nm1, nm1);
        *(uint2*)(dst + (int64_t)i * plane) = make_uint2(w0, w1);
      }
    }
  }
}

static int oz_slicev(const double2* x, int rows, int cols, int64_t batch, int64_t xstride, int s, const OzSliceOut& o,
                     cudaStream_t st) {
  const int ld = oz_ld(cols);
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int64_t nb = std::min<int64_t>(batch - b0, 65535);
    OzSliceOut ob = o;
    for (int q = 0; q < o.nc; ++q) {
      ob.sl[q] = o.sl[q] + b0 * (int64_t)s * rows * ld;
      ob.ex[q] = o.ex[q] + b0 * rows;
    }
    void* pr = prof_begin("oz_slice", st);
    const double2* xb = x + b0 * xstride;
    oz_rowexp_kernel<<<dim3((rows + 7) / 8, (unsigned)nb), 256, 0, st>>>(xb, rows, cols, xstride, ob);
    const int64_t groups = nb * rows * (int64_t)(ld / 8);
    static const int fpcut = getenv("QCH_OZ_FPCUT") ? atoi(getenv("QCH_OZ_FPCUT")) : 1;
    const int blocks = (int)std::min<int64_t>((groups + 255) / 256, (int64_t)sm_count() * 64);
    switch (s) {
#define OZ_SL(k) \
  case k: oz_cut_kernel<k><<<blocks, 256, 0, st>>>(xb, rows, cols, xstride, ob, groups, fpcut); break;
      OZ_SL(1) OZ_SL(2) OZ_SL(3) OZ_SL(4) OZ_SL(5) OZ_SL(6) OZ_SL(7) OZ_SL(8)
#undef OZ_SL
      default: return fail(QCH_ERR_VALUE, "ozaki: 1..8 slices");
    }
    prof_end(pr, st);
    QCH_LAUNCH_CHECK("oz_cut_kernel");
    note_launch(2);
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

// slices [planes][rows][ld] int8 as a 3-d map (columns beyond cols read as
// zeros), box 128 B x box_rows
static int oz_map(CUtensorMap* map, const int8_t* ptr, int64_t rows, int64_t cols, int64_t planes,
                  unsigned box_rows = 128) {
  auto fn = oz_encode();
  if (!fn) return fail(QCH_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int64_t ld = oz_ld((int)cols);
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)ld, (cuuint64_t)(rows * ld)};
  cuuint32_t box[3] = {(cuuint32_t)OZ_BK, (cuuint32_t)box_rows, 1u};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)ptr, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(QCH_ERR_CUDA, "cuTensorMapEncodeTiled (oz) failed (" + std::to_string((int)r) + ")");
  return QCH_OK;
}

int oz_slice(const double2* x, int rows, int cols, int64_t batch, int64_t xstride, int comp, int s, int8_t* sl, int* ex,
             cudaStream_t st) {
  OzSliceOut o{};
  o.sl[0] = sl;
  o.ex[0] = ex;
  o.comp[0] = comp;
  o.nc = 1;
  return oz_slicev(x, rows, cols, batch, xstride, s, o, st);
}

// P_b = X_b Y_b^T for a batch (slices as produced by oz_slice); tiles: null =
// all tiles, else a device list of ntiles (ti << 16 | tj)
// GEMM shape: 0 = 128 x 128 register accumulator (oz_gemm_kernel), 1 = 128 x
// 256 (one CTA), 2 = 256 x 128 (CTA pair), 3 = 256 x 256 (CTA pair; default)
// — QCH_OZ_CFG=r128 | w256 | p128 | p256
int oz_cfg() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("QCH_OZ_CFG");
    v = 3;
    if (e) {
      if (!strcmp(e, "r128")) v = 0;
      else if (!strcmp(e, "w256")) v = 1;
      else if (!strcmp(e, "p128")) v = 2;
    }
  }
  return v;
}
static int oz_tile_rows() { return oz_cfg() >= 2 ? 2 * OZ_BM : OZ_BM; }
static int oz_tile_cols() { return (oz_cfg() == 1 || oz_cfg() == 3) ? 256 : 128; }

template <int BN, bool PAIR>
static int oz_launch_w(const CUtensorMap& ma, const CUtensorMap& mb, const OzArgs& g, int64_t batch,
                       cudaStream_t st) {
  using W = OzW<BN, PAIR>;
  QCH_CUDA(smem_attr((const void*)oz_gemmw_kernel<BN, PAIR>, W::SMEM));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((PAIR ? 2 : 1) * g.ntiles, (unsigned)batch);
  cfg.blockDim = dim3(OZ_THREADS);
  cfg.dynamicSmemBytes = W::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = PAIR ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  QCH_CUDA(cudaLaunchKernelEx(&cfg, oz_gemmw_kernel<BN, PAIR>, ma, mb, g));
  return QCH_OK;
}

int oz_gemm(const int8_t* xs, const int* ea, const int8_t* ys, const int* eb, int m, int n, int k, int s,
            int64_t batch, double* out, int ldo, int64_t so, const int* tiles, int ntiles, cudaStream_t st,
            double* ops, int sp) {
  if (sp <= 0) sp = s;  // planes stored per item (the leading s of them are used: the digits of a shorter
                        // slicing are the leading digits of a longer one)
  if (s < 1 || s > OZ_MAX_S || s > sp) return fail(QCH_ERR_VALUE, "ozaki: 1..8 slices, at most the stored ones");
  if (ldo % 2 || ldo < n || so % 2) return fail(QCH_ERR_VALUE, "ozaki: the output row stride must be even and >= n");
  // exact int32 accumulation: (slices per diagonal) K 127^2 < 2^31
  if ((int64_t)s * k * 127 * 127 >= (int64_t)1 << 31)
    return fail(QCH_ERR_UNSUPPORTED, "ozaki: s K 127^2 must stay below 2^31");
  if (batch > 65535) return fail(QCH_ERR_UNSUPPORTED, "ozaki: batch > 65535");
  const int cfg = oz_cfg();
  const int rows_per_tile = oz_tile_rows(), bn = oz_tile_cols();
  CUtensorMap ma, mb;
  if (int rc = oz_map(&ma, xs, m, k, batch * sp)) return rc;
  if (int rc = oz_map(&mb, ys, n, k, batch * sp, cfg >= 2 ? bn / 2 : bn)) return rc;
  OzArgs g{};
  g.ea = ea;
  g.eb = eb;
  g.out = out;
  g.m = m;
  g.n = n;
  g.k = k;
  g.s = s;
  g.sp = sp;
  g.ldo = ldo;
  g.so = so;
  g.tiles = tiles;
  g.tn = (n + bn - 1) / bn;
  g.ntiles = tiles ? ntiles : ((m + rows_per_tile - 1) / rows_per_tile) * g.tn;
  if (ops) *ops = (double)g.ntiles * rows_per_tile * bn * (double)k * 2.0 * (s * (s + 1) / 2) * batch;
  void* pr = prof_begin("oz_gemm", st);
  int rc = QCH_OK;
  switch (cfg) {
    case 1: rc = oz_launch_w<256, false>(ma, mb, g, batch, st); break;
    case 2: rc = oz_launch_w<128, true>(ma, mb, g, batch, st); break;
    case 3: rc = oz_launch_w<256, true>(ma, mb, g, batch, st); break;
    default: {
      const int smem = OZ_ST * OZ_STAGE + 1024 + 256;
      QCH_CUDA(smem_attr((const void*)oz_gemm_kernel, smem));
      oz_gemm_kernel<<<dim3(g.ntiles, (unsigned)batch), OZ_THREADS, smem, st>>>(ma, mb, g);
    }
  }
  if (rc) return rc;
  QCH_LAUNCH_CHECK("oz_gemm_kernel");
  note_launch(1);
  prof_end(pr, st);
  return QCH_OK;
}

// C = A B for batches of Hermitian n x n A, B whose product is Hermitian
// (commuting Hermitian polynomials of one matrix), by the Gauss / 3M form on
// three Ozaki real products over the tiles meeting the lower triangle.  The
// Y operands are rows of B^T = conj(B) (Br symmetric, Bi antisymmetric):
//   P1 = Ar Br^T = Ar Br,  P2' = Ai Bi^T = -Ai Bi,  P3 = (Ar + Ai)(Br - Bi)^T
//   Re = P1 + P2',  Im = (P3 - P1) + P2'
// so A takes the components {Re, Im, Re + Im} and B {Re, Im, Re - Im}: a
// matrix used on both sides is sliced once into four.  The combine pass
// applies the epilogue (STORE / QACC / UFIN as zgemm_tma.cu) on the lower
// triangle and writes the mirror, 32 x 32 tile pairs through shared memory so
// both the tile and its transposed mirror are written coalesced.
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
  int ldp;  // row stride of P1..P3 (n rounded up to even)
  int tn;   // 32-tiles per side
};

__global__ void __launch_bounds__(256) oz_combine_kernel(OzCombine a) {
  __shared__ double2 mir[32][33];
  const int t = blockIdx.x;
  int I = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((I + 1) * (I + 2) / 2 <= t) ++I;
  while (I * (I + 1) / 2 > t) --I;
  const int J = t - I * (I + 1) / 2;
  const int64_t nn = (int64_t)a.n * a.n;
  const int64_t boff = (int64_t)blockIdx.y * nn;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = J * 32 + tx;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int rl = ty + 8 * k, r = I * 32 + rl;
    if (r >= a.n || c >= a.n || r < c) continue;
    const int64_t e = boff + (int64_t)r * a.n + c;
    const int64_t ep = (int64_t)blockIdx.y * a.n * a.ldp + (int64_t)r * a.ldp + c;
    const double v1 = a.p1[ep], v2 = a.p2[ep], v3 = a.p3[ep];
    const double re = v1 + v2, im = (v3 - v1) + v2;
    double2 d, m;
    if (a.mode == 3) {  // U = C - i S
      const double2 cv = a.pw[0][e];
      d = make_double2(cv.x + im, cv.y - re);
      m = make_double2(cv.x - im, -cv.y - re);
    } else {
      double xr = re, xi = im;
      if (a.mode == 2) {
        xr += (r == c) ? a.q[0] : 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (i < a.nq) {
            const double2 pv = a.pw[i][e];
            xr = fma(a.q[i + 1], pv.x, xr);
            xi = fma(a.q[i + 1], pv.y, xi);
          }
      }
      d = make_double2(xr, xi);
      m = make_double2(xr, -xi);
    }
    a.c[e] = d;
    mir[rl][tx] = m;
  }
  __syncthreads();
  // mirror: element (J*32 + rl', I*32 + tx') = mir[tx'][rl'] for r > c
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int cl = ty + 8 * k;           // local column of the lower tile = mirror row
    const int mr = J * 32 + cl, mc = I * 32 + tx;  // mirror position; source (r, c) = (mc, mr)
    if (mr >= a.n || mc >= a.n || mc <= mr) continue;
    a.c[boff + (int64_t)mr * a.n + mc] = mir[tx][cl];
  }
}

// tiles meeting the lower triangle (R rows x C columns as oz_cfg), in super-tiles of 1024 x 1024 so the ~148 concurrent CTAs share
// A and B slice panels (an L2-resident working set)
static int oz_lower_tiles(int n, const int** out, int* count, cudaStream_t st) {
  struct Key {
    int dev, n, r, c;
    bool operator<(const Key& o) const {
      return std::tie(dev, n, r, c) < std::tie(o.dev, o.n, o.r, o.c);
    }
  };
  static std::mutex mu;
  static std::map<Key, std::pair<int*, int>> lists;  // device tile lists, kept for the process
  const int R = oz_tile_rows(), C = oz_tile_cols();
  int dev = 0;
  QCH_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = lists.find(Key{dev, n, R, C});
  if (it == lists.end()) {
    const int TI = (n + R - 1) / R, TJ = (n + C - 1) / C;
    const int GI = 1024 / R, GJ = 1024 / C;
    std::vector<int> h;
    for (int bi = 0; bi < TI; bi += GI)
      for (int bj = 0; bj < TJ; bj += GJ)
        for (int i = bi; i < std::min(TI, bi + GI); ++i)
          for (int j = bj; j < std::min(TJ, bj + GJ); ++j)
            if (j * C <= i * R + R - 1) h.push_back((i << 16) | j);
    int* d = nullptr;
    QCH_CUDA(cudaMalloc((void**)&d, sizeof(int) * h.size()));
    QCH_CUDA(cudaMemcpyAsync(d, h.data(), sizeof(int) * h.size(), cudaMemcpyHostToDevice, st));
    QCH_CUDA(cudaStreamSynchronize(st));
    it = lists.emplace(Key{dev, n, R, C}, std::make_pair(d, (int)h.size())).first;
  }
  *out = it->second.first;
  *count = it->second.second;
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
static std::atomic<double> g_i8_fp64eq{0.0};  // complex-product flops (8 M N K, computed tiles) stood in for
double oz_int8_ops_total() { return g_i8_ops.load(); }
static void atomic_add_d(std::atomic<double>& a, double v) {
  double cur = a.load();
  while (!a.compare_exchange_weak(cur, cur + v)) {
  }
}

// ---- slice cache (OzCache, zgemm.h) ----
OzCache::~OzCache() { clear(); }

void OzCache::clear() {
  for (auto& e : ent)
    for (int q = 0; q < 4; ++q) {
      if (e.sl[q]) cudaFreeAsync(e.sl[q], st);
      if (e.ex[q]) cudaFreeAsync(e.ex[q], st);
    }
  ent.clear();
}

void OzCache::drop(const void* src) {
  for (size_t i = 0; i < ent.size(); ++i)
    if (ent[i].src == src) {
      for (int q = 0; q < 4; ++q) {
        if (ent[i].sl[q]) cudaFreeAsync(ent[i].sl[q], st);
        if (ent[i].ex[q]) cudaFreeAsync(ent[i].ex[q], st);
      }
      ent.erase(ent.begin() + (long)i);
      return;
    }
}

int OzCache::get(const double2* src, unsigned mask, const OzCache::Entry** out) {
  Entry* e = nullptr;
  for (auto& x : ent)
    if (x.src == src) e = &x;
  if (!e) {
    ent.push_back(Entry{});
    e = &ent.back();
    e->src = src;
  }
  const int S = oz_slices();
  const int64_t nn = (int64_t)n * n;
  OzSliceOut o{};
  for (int q = 0; q < 4; ++q)
    if ((mask >> q & 1) && !e->sl[q]) {
      QCH_CUDA(cudaMallocAsync((void**)&e->sl[q], (size_t)S * n * oz_ld(n) * batch, st));
      QCH_CUDA(cudaMallocAsync((void**)&e->ex[q], sizeof(int) * (size_t)n * batch, st));
      o.sl[o.nc] = e->sl[q];
      o.ex[o.nc] = e->ex[q];
      o.comp[o.nc] = q;
      ++o.nc;
    }
  if (o.nc)
    if (int rc = oz_slicev(src, n, n, batch, nn, S, o, st)) return rc;
  *out = e;
  return QCH_OK;
}

int zgemm_herm_ozaki(int mode, const double2* a, const double2* b, double2* c, const double2* const* pw,
                     const double* q, int nq, int n, int64_t batch, cudaStream_t st, OzCache* cache, int s_use) {
  if (c == a || c == b) return fail(QCH_ERR_VALUE, "ozaki Hermitian product: output aliases an operand");
  ensure_pool();
  OzCache local(n, batch, st);
  OzCache* oc = cache ? cache : &local;
  if (oc->n != n || oc->batch != batch) return fail(QCH_ERR_VALUE, "ozaki slice cache: shape mismatch");
  const int SP = oz_slices();                               // slices cut and stored
  const int S = (s_use > 0 && s_use < SP) ? s_use : SP;     // leading slices this product uses
  const int64_t nn = (int64_t)n * n;
  const OzCache::Entry *X = nullptr, *Y = nullptr;
  const unsigned ma = a == b ? 0xF : 0x7;  // A: Re, Im, Re + Im (+ Re - Im when it is also B)
  if (int rc = oc->get(a, ma, &X)) return rc;
  if (int rc = oc->get(b, 0xB, &Y)) return rc;  // B: Re, Im, Re - Im
  if (int rc = oc->get(a, ma, &X)) return rc;   // re-lookup (the entry vector may have grown)
  double* P = nullptr;
  const int ldp = (n + 1) & ~1;  // even: the GEMM epilogue's paired stores stay 16-byte aligned
  const int64_t np_ = (int64_t)n * ldp;
  QCH_CUDA(cudaMallocAsync((void**)&P, 3 * sizeof(double) * (size_t)np_ * batch, st));
  const int yc[3] = {0, 1, 3};
  int rc = QCH_OK;
  const int* tiles = nullptr;
  int ntiles = 0;
  rc = oz_lower_tiles(n, &tiles, &ntiles, st);
  double ops = 0.0;
  for (int v = 0; v < 3 && rc == QCH_OK; ++v) {
    double o = 0.0;
    rc = oz_gemm(X->sl[v], X->ex[v], Y->sl[yc[v]], Y->ex[yc[v]], n, n, n, S, batch, P + v * np_ * batch, ldp, np_, tiles,
                 ntiles, st, &o, SP);
    ops += o;
  }
  if (rc == QCH_OK) {
    atomic_add_d(g_i8_ops, ops);
    atomic_add_d(g_i8_fp64eq, 8.0 * ntiles * (double)oz_tile_rows() * oz_tile_cols() * n * batch);
    OzCombine cm{};
    cm.p1 = P;
    cm.p2 = P + np_ * batch;
    cm.p3 = P + 2 * np_ * batch;
    cm.c = c;
    cm.nq = nq;
    cm.mode = mode;
    cm.n = n;
    cm.ldp = ldp;
    cm.tn = (n + 31) / 32;
    for (int i = 0; i < 4; ++i) cm.pw[i] = (pw && i < (mode == 3 ? 1 : nq)) ? pw[i] : nullptr;
    for (int i = 0; i < 5; ++i) cm.q[i] = (q && i <= nq) ? q[i] : 0.0;
    const unsigned tiles32 = (unsigned)(cm.tn * (cm.tn + 1) / 2);
    for (int64_t b0 = 0; b0 < batch && rc == QCH_OK; b0 += 65535) {
      const int64_t nb = std::min<int64_t>(batch - b0, 65535);
      OzCombine cb = cm;
      cb.p1 += b0 * np_;
      cb.p2 += b0 * np_;
      cb.p3 += b0 * np_;
      cb.c += b0 * nn;
      for (int i = 0; i < 4; ++i)
        if (cb.pw[i]) cb.pw[i] += b0 * nn;
      void* pr = prof_begin("oz_combine", st);
      oz_combine_kernel<<<dim3(tiles32, (unsigned)nb), 256, 0, st>>>(cb);
      prof_end(pr, st);
      note_launch(1);
      if (cudaGetLastError() != cudaSuccess) rc = fail(QCH_ERR_CUDA, "oz_combine_kernel launch failed");
    }
  }
  cudaFreeAsync(P, st);
  oc->drop(c);  // c's cached slices (if any) are stale now
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
extern "C" double qch_int8_fp64_equiv_flops(void) { return g_i8_fp64eq.load(); }

// experimental: P (m x n, f64) = X Y^T for real components of complex matrices
// x (m x k) and y (n x k) (comp as oz_slice_kernel), s slices
extern "C" int qch_oz_real_test(const void* d_x, int xcomp, const void* d_y, int ycomp, void* d_out, int64_t m,
                                int64_t n, int64_t k, int s, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n % 2) return fail(QCH_ERR_VALUE, "qch_oz_real_test: n must be even (paired FP64 stores)");
  int8_t *xs = nullptr, *ys = nullptr;
  int *ea = nullptr, *eb = nullptr;
  ensure_pool();
  QCH_CUDA(cudaMallocAsync((void**)&xs, (size_t)s * m * oz_ld((int)k), st));
  QCH_CUDA(cudaMallocAsync((void**)&ys, (size_t)s * n * oz_ld((int)k), st));
  QCH_CUDA(cudaMallocAsync((void**)&ea, sizeof(int) * m, st));
  QCH_CUDA(cudaMallocAsync((void**)&eb, sizeof(int) * n, st));
  int rc = oz_slice((const double2*)d_x, (int)m, (int)k, 1, m * k, xcomp, s, xs, ea, st);
  if (!rc) rc = oz_slice((const double2*)d_y, (int)n, (int)k, 1, n * k, ycomp, s, ys, eb, st);
  if (!rc)
    rc = oz_gemm(xs, ea, ys, eb, (int)m, (int)n, (int)k, s, 1, (double*)d_out, (int)n, m * n, nullptr, 0, st, nullptr,
                 s);
  cudaFreeAsync(xs, st);
  cudaFreeAsync(ys, st);
  cudaFreeAsync(ea, st);
  cudaFreeAsync(eb, st);
  return rc;
}
