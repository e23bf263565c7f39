// zgemm_tma.cu — TMA-fed, warp-specialised DMMA complex128 GEMM (sm_100a).
//
// FP64 tensor work on sm_100a is the warp-level DMMA (mma.sync m8n8k4 f64 ->
// SASS DMMA.8x8x4; there is no tcgen05 kind::f64).  This kernel feeds it the
// Blackwell way: one producer warp streams the operand tiles with TMA
// (cp.async.bulk.tensor, SASS UTMALDG) into a 6-stage shared-memory ring with
// full/empty mbarriers; eight consumer warps (32x32 complex each, CTA tile
// 128x64) run the DMMAs and never touch a block barrier.  Persistent: one CTA
// per SM walks the tiles, the producer running ahead into the next tile while
// the consumers finish the previous one's epilogue.
//
// Layout.  complex128 stays interleaved: the tensor maps are over float64
// with the inner dimension doubled; a box is 16 doubles (8 complex, 128 B)
// wide and the maps use the 128-byte swizzle (16-byte chunk c of 128-byte
// smem line r lands at chunk c ^ (r & 7)).
//   A tile  : rows m0..m0+127, complex k0..k0+7 -> 128 lines of 128 B.
//   B tile  : (k-major) 8 boxes of 8 k-rows x 8 complex columns -> box g
//             holds columns n0+8g..+7; (BH, B = conj(Bm)^T) rows n of Bm,
//             like A.
// DMMA k-slot permutation: DMMA step kk in {0,1} of a stage pairs its four
// k slots with complex columns {kk, kk+2, kk+4, kk+6}.  With the swizzle this
// makes every 8-lane phase of a fragment LDS.128 hit 8 distinct 16-byte bank
// groups (conflict free, no padding), for A, B and BH alike.
//
// Complex product: by default THREE real DMMA products (Gauss / 3M):
//     P1 = Ar Br, P2 = Ai Bi, P3 = (Ar + Ai)(Br + Bi);  Re = P1 - P2,
//     Im = P3 - P1 - P2
// (6 N^3 DMMA flops per complex GEMM instead of 8 N^3; the error bound
// grows from eps |A||B| componentwise to eps (|Ar|+|Ai|)(|Br|+|Bi|), ~1e-14
// relative here — the parity bar is 1e-10).  QCH_ZGEMM_3M=0: four products,
// Cr += Ar Br + (-Ai) Bi, Ci += Ar Bi + Ai Br.
//
// Epilogues (fused):
//   STORE   C = A B
//   ACCUM   C += A B
//   QACC    C = q0 I + sum_{i=1..nq} q_i P_i + A B     (Paterson-Stockmeyer
//           Horner step with the Q_j formation fused)
//   UFIN    U = C - i (A B)   (exp(-iH) = cos H - i sin H, last step)
//   DEFECT  acc[b] += || A A^H - I ||_F^2  (BH; unitarity audit)
// HERM: the product is known to be Hermitian (both factors are Hermitian
// polynomials of one matrix, or A A^H): only the tiles meeting the lower
// triangle are computed; element (r, c) is written for r >= c, and for r > c
// also its mirror (c, r) = conj (DEFECT: r > c counts twice) — about half
// the DMMA work.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>

#include "zgemm.h"

namespace qch {

constexpr int ZT_BM = 128, ZT_BN = 64, ZT_BK = 8, ZT_ST = 6;
constexpr int ZT_ABYTES = ZT_BM * ZT_BK * 16;  // 16 KB
constexpr int ZT_BBYTES = ZT_BN * ZT_BK * 16;  // 8 KB
constexpr int ZT_STAGE = ZT_ABYTES + ZT_BBYTES;
constexpr int ZT_CONSUMERS = 8;    // 2 warpgroups: 4 (m) x 2 (n) warps of 32x32
constexpr int ZT_THREADS = 384;    // + 1 producer warpgroup (one TMA lane); registers
                                   // moved to the consumers with setmaxnreg

__device__ __forceinline__ unsigned zt_smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void zt_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n ZT_W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra ZT_W;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void zt_tma3(unsigned dst, const CUtensorMap* map, int c0, int c1, int c2, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void zt_dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// tile t (of the per-matrix tile list) -> (ti, tj) in units of (ZT_BM, ZT_BN)
__device__ __forceinline__ void zt_tile(int t, const ZtArgs& g, bool herm, int& ti, int& tj) {
  if (herm) {  // tiles meeting the lower triangle: row ti holds tiles tj = 0 .. 2 ti + 1 (clipped to tn)
    int r = 0, acc = 0;
    for (;; ++r) {
      const int cnt = min(2 * r + 2, g.tn);
      if (t < acc + cnt) break;
      acc += cnt;
    }
    ti = r;
    tj = t - acc;
  } else {  // bands of 8 tile rows, column-major inside a band (L2 reuse)
    const int band = t / (8 * g.tn);
    const int rows = min(8, g.tm - band * 8);
    const int idx = t - band * 8 * g.tn;
    ti = band * 8 + idx % rows;
    tj = idx / rows;
  }
}

template <int MODE, bool HERM, bool BH, bool M3>
__global__ void __launch_bounds__(ZT_THREADS, 1)
    zgemm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, ZtArgs g) {
  extern __shared__ unsigned char zt_raw[];
  unsigned char* base = (unsigned char*)(((uintptr_t)zt_raw + 1023) & ~(uintptr_t)1023);
  unsigned long long* full = (unsigned long long*)(base + ZT_ST * ZT_STAGE);
  unsigned long long* empty = full + ZT_ST;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KT = (g.k + ZT_BK - 1) / ZT_BK;
  const int64_t total = (int64_t)g.tiles * g.nbatch;  // (batch item, tile) pairs of this launch

  if (tid == 0) {
    for (int s = 0; s < ZT_ST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(zt_smem_u32(full + s)) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(zt_smem_u32(empty + s)), "r"(ZT_CONSUMERS)
                   : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp >= ZT_CONSUMERS) {  // ===== producer warpgroup: one TMA lane, runs ahead across tiles
    asm volatile("setmaxnreg.dec.sync.aligned.u32 24;" ::: "memory");
    if (warp == ZT_CONSUMERS && lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
      int it = 0;
      for (int64_t w = blockIdx.x; w < total; w += gridDim.x) {
        const int bz = (int)(g.b0 + w / g.tiles);
        int ti, tj;
        zt_tile((int)(w % g.tiles), g, HERM, ti, tj);
        const int m0 = ti * ZT_BM, n0 = tj * ZT_BN;
        for (int kt = 0; kt < KT; ++kt, ++it) {
          const int s = it % ZT_ST;
          zt_wait(zt_smem_u32(empty + s), (unsigned)(((it / ZT_ST) & 1) ^ 1));
          const unsigned fb = zt_smem_u32(full + s);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(ZT_STAGE) : "memory");
          const unsigned dA = zt_smem_u32(base + s * ZT_STAGE);
          const unsigned dB = dA + ZT_ABYTES;
          zt_tma3(dA, &tmA, 2 * kt * ZT_BK, m0, bz, fb);
          if (BH) {
            zt_tma3(dB, &tmB, 2 * kt * ZT_BK, n0, bz, fb);
          } else {
#pragma unroll
            for (int q = 0; q < ZT_BN / 8; ++q)
              zt_tma3(dB + q * 1024, &tmB, 2 * (n0 + 8 * q), kt * ZT_BK, bz, fb);
          }
        }
      }
    }
    return;
  }

  // ===== consumers: warp (wm, wn) owns rows wm*32.., cols wn*32.. of the tile
  asm volatile("setmaxnreg.inc.sync.aligned.u32 240;" ::: "memory");
  const int wm = warp & 3, wn = warp >> 2;
  const int fr = lane >> 2, fk = lane & 3;
  int it = 0;
  for (int64_t w = blockIdx.x; w < total; w += gridDim.x) {
    const int64_t bz = g.b0 + w / g.tiles;
    int ti, tj;
    zt_tile((int)(w % g.tiles), g, HERM, ti, tj);
    const int m0 = ti * ZT_BM, n0 = tj * ZT_BN;
    // 4M: cr = Re, ci = Im.  M3 (Gauss): cr = Ar Br, p2 = Ai Bi,
    // ci = (Ar + Ai)(Br + Bi) -> Re = cr - p2, Im = ci - cr - p2 (3 DMMAs
    // per complex product instead of 4)
    double cr[4][4][2], ci[4][4][2], p2[M3 ? 4 : 1][4][2];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        cr[x][y][0] = cr[x][y][1] = 0.0;
        ci[x][y][0] = ci[x][y][1] = 0.0;
        if (M3) p2[M3 ? x : 0][y][0] = p2[M3 ? x : 0][y][1] = 0.0;
      }
    for (int kt = 0; kt < KT; ++kt, ++it) {
      const int s = it % ZT_ST;
      zt_wait(zt_smem_u32(full + s), (unsigned)((it / ZT_ST) & 1));
      const unsigned char* As = base + s * ZT_STAGE;
      const unsigned char* Bs = As + ZT_ABYTES;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const int kl = 2 * fk + kk;  // complex column of this lane's k slot
        // B fragments of the 4 column tiles stay live; A fragments are loaded
        // one row tile at a time
        double br[4], bi[4], bs[4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          double2 v;
          if (BH) {
            const int row = wn * 32 + nt * 8 + fr;
            v = *(const double2*)(Bs + row * 128 + ((kl ^ fr) << 4));
            v.y = -v.y;
          } else {
            v = *(const double2*)(Bs + (wn * 4 + nt) * 1024 + kl * 128 + ((fr ^ kl) << 4));
          }
          br[nt] = v.x;
          bi[nt] = v.y;
          if (M3) bs[nt] = v.x + v.y;
        }
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          const int row = wm * 32 + mt * 8 + fr;
          const double2 v = *(const double2*)(As + row * 128 + ((kl ^ fr) << 4));
          const double ar = v.x, ai = v.y;
          if (M3) {
            const double as = v.x + v.y;
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
              zt_dmma(cr[mt][nt][0], cr[mt][nt][1], ar, br[nt]);
              zt_dmma(p2[M3 ? mt : 0][nt][0], p2[M3 ? mt : 0][nt][1], ai, bi[nt]);
              zt_dmma(ci[mt][nt][0], ci[mt][nt][1], as, bs[nt]);
            }
          } else {
            const double nai = -v.y;
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
              zt_dmma(cr[mt][nt][0], cr[mt][nt][1], ar, br[nt]);
              zt_dmma(ci[mt][nt][0], ci[mt][nt][1], ar, bi[nt]);
              zt_dmma(cr[mt][nt][0], cr[mt][nt][1], nai, bi[nt]);
              zt_dmma(ci[mt][nt][0], ci[mt][nt][1], ai, br[nt]);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(zt_smem_u32(empty + s)) : "memory");
    }

    // ===== epilogue: lane owns C[row][2 fk + e] of each 8x8 sub-tile.  HERM:
    // write r >= c only, with the mirror (c, r) = conj for r > c.
    double dsum = 0.0;
    const int64_t cb = bz * g.sc;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int r = m0 + wm * 32 + mt * 8 + fr;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = n0 + wn * 32 + nt * 8 + 2 * fk + e;
          if (r >= g.m || c >= g.n) continue;
          if (HERM && r < c) continue;
          const bool mirror = HERM && r > c;
          double re = cr[mt][nt][e], im = ci[mt][nt][e];
          if (M3) {
            const double q2 = p2[M3 ? mt : 0][nt][e];
            im = (im - re) - q2;
            re = re - q2;
          }
          const int64_t off = cb + (int64_t)r * g.ldc + c;
          const int64_t moff = cb + (int64_t)c * g.ldc + r;
          if (MODE == ZT_DEFECT) {
            const double dr = re - (r == c ? 1.0 : 0.0);
            dsum += (mirror ? 2.0 : 1.0) * (dr * dr + im * im);
            continue;
          }
          double2 v;
          if (MODE == ZT_STORE) {
            v = make_double2(re, im);
          } else if (MODE == ZT_ACCUM) {
            const double2 o = g.c[off];
            v = make_double2(o.x + re, o.y + im);
          } else if (MODE == ZT_QACC) {
            double xr = (r == c) ? g.q[0] : 0.0, xi = 0.0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (i < g.nq) {
                const double2 pv = g.p[i][off];
                xr = fma(g.q[i + 1], pv.x, xr);
                xi = fma(g.q[i + 1], pv.y, xi);
              }
            v = make_double2(xr + re, xi + im);
          } else {  // UFIN: U = C - i S,  S = (re, im)
            const double2 cv = g.p[0][off];
            g.c[off] = make_double2(cv.x + im, cv.y - re);
            if (mirror) g.c[moff] = make_double2(cv.x - im, -cv.y - re);
            continue;
          }
          g.c[off] = v;
          if (mirror) g.c[moff] = make_double2(v.x, -v.y);
        }
      }
    }
    if (MODE == ZT_DEFECT) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, off);
      if (lane == 0) atomicAdd(g.acc + bz, dsum);
    }
  }
}

// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// 3-d map over a batch of row-major complex matrices (rows x cols, batch
// stride in complex elements) viewed as float64 [batch][rows][2 cols]; box =
// 8 complex x box_rows, 128-byte swizzle.
static int zt_map(CUtensorMap* map, const double2* ptr, int64_t rows, int64_t cols, int64_t batch, int64_t stride,
                  int box_rows) {
  auto fn = encode_fn();
  if (!fn) return fail(QCH_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)(2 * cols), (cuuint64_t)rows, (cuuint64_t)std::max<int64_t>(batch, 1)};
  cuuint64_t strides[2] = {(cuuint64_t)(cols * 16), (cuuint64_t)(std::max<int64_t>(stride, rows * cols) * 16)};
  cuuint32_t box[3] = {16, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)ptr, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(QCH_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return QCH_OK;
}

static const char* zt_name(int mode, bool herm) {
  switch (mode) {
    case ZT_STORE: return herm ? "zgemm_herm" : "zgemm";
    case ZT_ACCUM: return "zgemm_accum";
    case ZT_QACC: return herm ? "zgemm_herm_qacc" : "zgemm_qacc";
    case ZT_UFIN: return "zgemm_herm_ufin";
    default: return herm ? "zgemm_herm_defect" : "zgemm_defect";
  }
}

// executed DMMA flops of every launch (roofline accounting, qch_dmma_flops):
// computed tiles x 128 x 64 complex outputs x K x (2 x real products)
static std::atomic<double> g_dmma_flops{0.0};
double dmma_flops_total() { return g_dmma_flops.load(); }

template <int MODE, bool HERM, bool BH, bool M3>
static int zt_launch(const CUtensorMap& ma, const CUtensorMap& mb, ZtArgs g, int64_t batch, cudaStream_t st) {
  const int smem = ZT_ST * ZT_STAGE + 2 * ZT_ST * 8 + 1024;
  QCH_CUDA(smem_attr((const void*)zgemm_tma_kernel<MODE, HERM, BH, M3>, smem));
  g.tm = (g.m + ZT_BM - 1) / ZT_BM;
  g.tn = (g.n + ZT_BN - 1) / ZT_BN;
  if (HERM) {
    g.tiles = 0;
    for (int r = 0; r < g.tm; ++r) g.tiles += std::min(2 * r + 2, g.tn);
  } else {
    g.tiles = g.tm * g.tn;
  }
  void* pr = prof_begin(zt_name(MODE, HERM), st);
  const int64_t per = std::max<int64_t>(1, (int64_t)(1u << 30) / g.tiles);  // work items per launch < 2^30
  for (int64_t done = 0; done < batch; done += per) {
    g.b0 = done;
    g.nbatch = (int)std::min<int64_t>(batch - done, per);
    const int64_t work = (int64_t)g.tiles * g.nbatch;
    const int grid = (int)std::min<int64_t>(work, sm_count());  // persistent: one CTA per SM
    {
      const double f = (double)work * ZT_BM * ZT_BN * (double)g.k * 2.0 * (M3 ? 3.0 : 4.0);
      double cur = g_dmma_flops.load();
      while (!g_dmma_flops.compare_exchange_weak(cur, cur + f)) {
      }
    }
    zgemm_tma_kernel<MODE, HERM, BH, M3><<<grid, ZT_THREADS, smem, st>>>(ma, mb, g);
    QCH_LAUNCH_CHECK("zgemm_tma_kernel");
    note_launch(1);
  }
  prof_end(pr, st);
  return QCH_OK;
}

// 3 real DMMA products per complex product (Gauss / 3M) by default;
// QCH_ZGEMM_3M=0 selects the 4-product form.
bool zgemm_use_3m() {
  static const bool v = [] {
    const char* e = getenv("QCH_ZGEMM_3M");
    return e == nullptr || atoi(e) != 0;
  }();
  return v;
}

// Generic entry: C (m x n) = op(A (m x k) B (k x n)) for a contiguous batch.
// herm requires m == n (and a Hermitian result); bh: B given as Bm (n x k),
// used as conj(Bm)^T.
int zt_gemm(int mode, bool herm, bool bh, const double2* a, const double2* b, int m, int n, int k, int64_t batch,
            int64_t sa, int64_t sb, ZtArgs g, cudaStream_t st) {
  if (batch <= 0 || m <= 0 || n <= 0 || k <= 0) return QCH_OK;
  if (batch > INT32_MAX) return fail(QCH_ERR_UNSUPPORTED, "zgemm: batch too large");
  CUtensorMap ma, mb;
  if (int rc = zt_map(&ma, a, m, k, batch, sa, ZT_BM)) return rc;
  if (bh) {
    if (int rc = zt_map(&mb, b, n, k, batch, sb, ZT_BN)) return rc;
  } else {
    if (int rc = zt_map(&mb, b, k, n, batch, sb, 8)) return rc;
  }
  g.m = m;
  g.n = n;
  g.k = k;
  if (g.ldc == 0) g.ldc = n;
  if (g.sc == 0) g.sc = (int64_t)m * n;
  const bool m3 = zgemm_use_3m();
#define ZT_CASE(MD, H, B)                                                                          \
  if (mode == MD && herm == H && bh == B)                                                          \
    return m3 ? zt_launch<MD, H, B, true>(ma, mb, g, batch, st) : zt_launch<MD, H, B, false>(ma, mb, g, batch, st);
  ZT_CASE(ZT_STORE, false, false)
  ZT_CASE(ZT_STORE, true, false)
  ZT_CASE(ZT_ACCUM, false, false)
  ZT_CASE(ZT_QACC, false, false)
  ZT_CASE(ZT_QACC, true, false)
  ZT_CASE(ZT_UFIN, true, false)
  ZT_CASE(ZT_DEFECT, true, true)
  ZT_CASE(ZT_DEFECT, false, true)
#undef ZT_CASE
  return fail(QCH_ERR_UNSUPPORTED, "zgemm: unsupported mode combination");
}

}  // namespace qch
