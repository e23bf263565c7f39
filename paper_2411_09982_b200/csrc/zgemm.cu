// zgemm.cu — the round-1 cp.async DMMA GEMM (kept for A/B comparison with
// QCH_ZGEMM=cpasync) and the dispatchers onto the TMA kernel (zgemm_tma.cu),
// the default.
//
// sm_100a has no tcgen05 kind::f64, so FP64 tensor work is the warp-level
// DMMA (mma.sync.aligned.m8n8k4 f64 -> SASS DMMA.8x8x4).  Complex operands stay
// interleaved (numpy complex128) in global AND shared memory: one 16-byte LDS
// fetches the (re, im) pair a fragment lane needs, so no de-interleave pass is
// spent.  A complex tile product is four real DMMA products:
//     Cr += Ar*Br + (-Ai)*Bi,   Ci += Ar*Bi + Ai*Br.
// Tiles: CTA 64x64 complex, BK = 8 complex, 4 warps of 32x32, 3-stage cp.async
// pipeline (16-byte cp.async.cg, zero-filled at the edges).  Shared-memory rows
// are padded so every quarter-warp fragment load is bank-conflict free.
//
// Epilogues (fused, no extra pass over C):
//   STORE   C = A op(B)
//   DEFECT  sum |(A B^H) - I|^2 into a per-batch accumulator (unitarity audit,
//           npad.py:257, expm.py:35-38)
//   ACCUM   C += A B   (Paterson-Stockmeyer Horner steps of exp(-iH))
#include "zgemm.h"
#include <cstring>
#include "qch_math.cuh"

namespace qch {

enum { ZG_STORE = 0, ZG_DEFECT = 2, ZG_ACCUM = 3 };

struct ZgemmArgs {
  const double2* a;
  const double2* b;
  double2* c;   // STORE / ACCUM: C
  double* acc;  // DEFECT: per-batch sum of squares
  int m, n, k;
  int64_t sa, sb, sc;  // batch strides (elements)
  int lda, ldb, ldc;
};

constexpr int BM = 64, BN = 64, BK = 8, STAGES = 3;
constexpr int APAD = 4;  // complex elements of padding per A row (64 B)
constexpr int BPAD = 2;  // per B row in k-major layout (32 B)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int MODE, bool BH>
__global__ void __launch_bounds__(128) zgemm_kernel(ZgemmArgs g) {
  // A tile [BM][BK+APAD]; B tile k-major [BK][BN+BPAD] or (BH) n-major [BN][BK+APAD]
  constexpr int A_ELEMS = BM * (BK + APAD);
  constexpr int B_ELEMS = BH ? BN * (BK + APAD) : BK * (BN + BPAD);
  extern __shared__ __align__(16) double2 zsm[];
  double2* As = zsm;
  double2* Bs = zsm + STAGES * A_ELEMS;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int64_t bz = blockIdx.z;
  const double2* __restrict__ A = g.a + bz * g.sa;
  const double2* __restrict__ B = g.b + bz * g.sb;
  const int KT = (g.k + BK - 1) / BK;

  auto load_stage = [&](int st, int kt) {
    const int k0 = kt * BK;
    double2* as = As + st * A_ELEMS;
    double2* bs = Bs + st * B_ELEMS;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int idx = tid + q * 128;
      int r = idx >> 3, cc = idx & 7;
      int gr = m0 + r, gk = k0 + cc;
      bool p = gr < g.m && gk < g.k;
      const double2* src = p ? A + (int64_t)gr * g.lda + gk : A;
      cp_async16(as + r * (BK + APAD) + cc, src, p);
    }
    if (BH) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int idx = tid + q * 128;
        int r = idx >> 3, cc = idx & 7;  // r = n, cc = k
        int gn = n0 + r, gk = k0 + cc;
        bool p = gn < g.n && gk < g.k;
        const double2* src = p ? B + (int64_t)gn * g.ldb + gk : B;
        cp_async16(bs + r * (BK + APAD) + cc, src, p);
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int idx = tid + q * 128;
        int r = idx >> 6, cc = idx & 63;  // r = k, cc = n
        int gk = k0 + r, gn = n0 + cc;
        bool p = gk < g.k && gn < g.n;
        const double2* src = p ? B + (int64_t)gk * g.ldb + gn : B;
        cp_async16(bs + r * (BN + BPAD) + cc, src, p);
      }
    }
  };

  double cr[4][4][2], ci[4][4][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      cr[x][y][0] = cr[x][y][1] = 0.0;
      ci[x][y][0] = ci[x][y][1] = 0.0;
    }

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_commit();
  }

  const int fr = lane >> 2, fk = lane & 3;
  for (int kt = 0; kt < KT; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    const int st = kt % STAGES;
    const double2* as = As + st * A_ELEMS;
    const double2* bs = Bs + st * B_ELEMS;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double ar[4], ai[4], nai[4], br[4], bi[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        double2 v = as[(wm * 32 + mt * 8 + fr) * (BK + APAD) + kk + fk];
        ar[mt] = v.x;
        ai[mt] = v.y;
        nai[mt] = -v.y;
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        double2 v;
        if (BH) {
          v = bs[(wn * 32 + nt * 8 + fr) * (BK + APAD) + kk + fk];
          v.y = -v.y;
        } else {
          v = bs[(kk + fk) * (BN + BPAD) + wn * 32 + nt * 8 + fr];
        }
        br[nt] = v.x;
        bi[nt] = v.y;
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          dmma(cr[mt][nt][0], cr[mt][nt][1], ar[mt], br[nt]);
          dmma(ci[mt][nt][0], ci[mt][nt][1], ar[mt], bi[nt]);
          dmma(cr[mt][nt][0], cr[mt][nt][1], nai[mt], bi[nt]);
          dmma(ci[mt][nt][0], ci[mt][nt][1], ai[mt], br[nt]);
        }
    }
    const int nk = kt + STAGES - 1;
    if (nk < KT) load_stage(nk % STAGES, nk);
    cp_commit();
  }
  cp_wait<0>();

  // epilogue: lane owns C[row][2*fk + {0,1}] of each 8x8 tile
  double dsum = 0.0;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int r = m0 + wm * 32 + mt * 8 + fr;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cidx = n0 + wn * 32 + nt * 8 + 2 * fk + e;
        if (r >= g.m || cidx >= g.n) continue;
        double re = cr[mt][nt][e], im = ci[mt][nt][e];
        const int64_t off = bz * g.sc + (int64_t)r * g.ldc + cidx;
        if (MODE == ZG_STORE) {
          g.c[off] = make_double2(re, im);
        } else if (MODE == ZG_ACCUM) {
          const double2 o = g.c[off];
          g.c[off] = make_double2(o.x + re, o.y + im);
        } else {
          double dr = re - (r == cidx ? 1.0 : 0.0);
          dsum += dr * dr + im * im;
        }
      }
    }
  }
  if (MODE == ZG_DEFECT) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, off);
    if (lane == 0) atomicAdd(g.acc + bz, dsum);
  }
}

static size_t zgemm_smem(bool bh) {
  size_t a = (size_t)BM * (BK + APAD);
  size_t b = bh ? (size_t)BN * (BK + APAD) : (size_t)BK * (BN + BPAD);
  return STAGES * (a + b) * sizeof(double2);
}

template <int MODE, bool BH>
static int zgemm_launch(const ZgemmArgs& g, int64_t batch, cudaStream_t st) {
  size_t smem = zgemm_smem(BH);
  QCH_CUDA(smem_attr((const void*)zgemm_kernel<MODE, BH>, (int)smem));
  int64_t done = 0;
  while (done < batch) {  // gridDim.z <= 65535
    int64_t nb = std::min<int64_t>(batch - done, 65535);
    ZgemmArgs h = g;
    h.a += done * g.sa;
    h.b += done * g.sb;
    if (h.c) h.c += done * g.sc;
    if (h.acc) h.acc += done;
    dim3 grid((g.n + BN - 1) / BN, (g.m + BM - 1) / BM, (unsigned)nb);
    void* pr = prof_begin(MODE == ZG_STORE    ? "zgemm"
                          : MODE == ZG_ACCUM  ? "zgemm_accum"
                                              : "zgemm_defect",
                          st);
    zgemm_kernel<MODE, BH><<<grid, 128, smem, st>>>(h);
    prof_end(pr, st);
    QCH_LAUNCH_CHECK("zgemm_kernel");
    note_launch(1);
    done += nb;
  }
  return QCH_OK;
}

// The TMA-fed kernel (zgemm_tma.cu) is the default; QCH_ZGEMM=cpasync selects
// this file's cp.async kernel (A/B comparisons).
static bool use_cpasync() {
  static const int v = [] {
    const char* e = getenv("QCH_ZGEMM");
    return (e && strcmp(e, "cpasync") == 0) ? 1 : 0;
  }();
  return v != 0;
}

// C = A @ B (square/rect, batched, contiguous)
static int zgemm_cpasync(const double2* a, const double2* b, double2* c, int m, int n, int k, int64_t batch, int64_t sa, int64_t sb,
          int64_t sc, cudaStream_t st) {
  ZgemmArgs g{};
  g.a = a;
  g.b = b;
  g.c = c;
  g.m = m;
  g.n = n;
  g.k = k;
  g.sa = sa;
  g.sb = sb;
  g.sc = sc;
  g.lda = k;
  g.ldb = n;
  g.ldc = n;
  return zgemm_launch<ZG_STORE, false>(g, batch, st);
}

// C += A @ B   (square n x n, batched contiguous; C must not alias A or B)
static int zgemm_accum_cpasync(const double2* a, const double2* b, double2* c, int n, int64_t batch, cudaStream_t st) {
  ZgemmArgs g{};
  g.a = a;
  g.b = b;
  g.c = c;
  g.m = g.n = g.k = n;
  g.sa = g.sb = g.sc = (int64_t)n * n;
  g.lda = g.ldb = g.ldc = n;
  return zgemm_launch<ZG_ACCUM, false>(g, batch, st);
}

// acc[b] += || U_b U_b^H - I ||_F^2
static int zgemm_defect_cpasync(const double2* u, double* acc, int n, int64_t batch, cudaStream_t st) {
  ZgemmArgs g{};
  g.a = u;
  g.b = u;
  g.acc = acc;
  g.m = g.n = g.k = n;
  g.sa = g.sb = (int64_t)n * n;
  g.sc = 0;
  g.lda = g.ldb = n;
  g.ldc = n;
  return zgemm_launch<ZG_DEFECT, true>(g, batch, st);
}

// ---- dispatch: TMA kernel (default) or the cp.async kernel above
int zgemm(const double2* a, const double2* b, double2* c, int m, int n, int k, int64_t batch, int64_t sa, int64_t sb,
          int64_t sc, cudaStream_t st) {
  if (use_cpasync()) return zgemm_cpasync(a, b, c, m, n, k, batch, sa, sb, sc, st);
  ZtArgs g{};
  g.c = c;
  g.sc = sc;
  return zt_gemm(ZT_STORE, false, false, a, b, m, n, k, batch, sa, sb, g, st);
}

int zgemm_accum(const double2* a, const double2* b, double2* c, int n, int64_t batch, cudaStream_t st) {
  if (use_cpasync()) return zgemm_accum_cpasync(a, b, c, n, batch, st);
  ZtArgs g{};
  g.c = c;
  const int64_t nn = (int64_t)n * n;
  return zt_gemm(ZT_ACCUM, false, false, a, b, n, n, n, batch, nn, nn, g, st);
}

// acc[b] += || U_b U_b^H - I ||_F^2 ; U U^H is Hermitian: lower tiles only
int zgemm_defect(const double2* u, double* acc, int n, int64_t batch, cudaStream_t st) {
  if (use_cpasync()) return zgemm_defect_cpasync(u, acc, n, batch, st);
  ZtArgs g{};
  g.acc = acc;
  const int64_t nn = (int64_t)n * n;
  return zt_gemm(ZT_DEFECT, true, true, u, u, n, n, n, batch, nn, nn, g, st);
}

// Hermitian products of the exp(-iH) evaluation: Ozaki-sliced int8 tcgen05
// GEMMs (ozgemm.cu) for 512 <= n <= 16384 by default, the DMMA kernel
// otherwise or with QCH_HERM_GEMM=dmma
static thread_local int t_herm_force_dmma = 0;
void herm_force_dmma(bool on) { t_herm_force_dmma = on ? 1 : 0; }
static int oz_min_n() {
  static const int v = getenv("QCH_OZ_MIN_N") ? std::max(16, atoi(getenv("QCH_OZ_MIN_N"))) : 512;
  return v;
}
bool herm_use_ozaki(int n) { return herm_engine() != 0 && !t_herm_force_dmma && n >= oz_min_n() && n <= 16384; }
static bool use_ozaki(int n) { return herm_use_ozaki(n); }

int zgemm_herm(const double2* a, const double2* b, double2* c, int n, int64_t batch, cudaStream_t st, OzCache* oc,
               int s_use) {
  if (use_ozaki(n)) return zgemm_herm_ozaki(ZT_STORE, a, b, c, nullptr, nullptr, 0, n, batch, st, oc, s_use);
  ZtArgs g{};
  g.c = c;
  const int64_t nn = (int64_t)n * n;
  return zt_gemm(ZT_STORE, true, false, a, b, n, n, n, batch, nn, nn, g, st);
}

int zgemm_qacc(bool herm, const double2* a, const double2* b, double2* c, const double2* const* p, const double* q,
               int nq, int n, int64_t batch, cudaStream_t st, OzCache* oc, int s_use) {
  if (nq > 4) return fail(QCH_ERR_UNSUPPORTED, "zgemm_qacc: at most 4 power terms");
  if (herm && use_ozaki(n)) return zgemm_herm_ozaki(ZT_QACC, a, b, c, p, q, nq, n, batch, st, oc, s_use);
  ZtArgs g{};
  g.c = c;
  g.nq = nq;
  g.q[0] = q[0];
  for (int i = 0; i < nq; ++i) {
    g.p[i] = p[i];
    g.q[i + 1] = q[i + 1];
  }
  const int64_t nn = (int64_t)n * n;
  return zt_gemm(ZT_QACC, herm, false, a, b, n, n, n, batch, nn, nn, g, st);
}

int zgemm_ufin(const double2* a, const double2* b, const double2* cpart, double2* u, int n, int64_t batch,
               cudaStream_t st, OzCache* oc, int s_use) {
  if (use_ozaki(n)) {
    const double2* pw[1] = {cpart};
    return zgemm_herm_ozaki(ZT_UFIN, a, b, u, pw, nullptr, 0, n, batch, st, oc, s_use);
  }
  ZtArgs g{};
  g.c = u;
  g.p[0] = cpart;
  const int64_t nn = (int64_t)n * n;
  return zt_gemm(ZT_UFIN, true, false, a, b, n, n, n, batch, nn, nn, g, st);
}

__global__ void sqrt_kernel(double* x, int64_t n) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < n) x[k] = sqrt(x[k]);
}

}  // namespace qch

using namespace qch;

extern "C" int qch_zgemm_batched(const void* d_a, const void* d_b, void* d_c, int64_t m, int64_t n, int64_t k,
                                 int64_t batch, int64_t stride_a, int64_t stride_b, int64_t stride_c, void* stream) {
  if (m <= 0 || n <= 0 || k <= 0 || batch <= 0) return QCH_OK;
  if (m > INT32_MAX / 2 || n > INT32_MAX / 2 || k > INT32_MAX / 2) return fail(QCH_ERR_UNSUPPORTED, "zgemm: too large");
  return zgemm((const double2*)d_a, (const double2*)d_b, (double2*)d_c, (int)m, (int)n, (int)k, batch, stride_a,
               stride_b, stride_c, (cudaStream_t)stream);
}

extern "C" int qch_zgemm_real_products(void) { return zgemm_use_3m() ? 3 : 4; }

extern "C" double qch_dmma_flops(void) { return dmma_flops_total(); }

extern "C" int qch_zgemm_herm_batched(const void* d_a, const void* d_b, void* d_c, int64_t n, int64_t batch,
                                      void* stream) {
  if (n <= 0 || batch <= 0) return QCH_OK;
  if (n > INT32_MAX / 2) return fail(QCH_ERR_UNSUPPORTED, "zgemm: too large");
  return zgemm_herm((const double2*)d_a, (const double2*)d_b, (double2*)d_c, (int)n, batch, (cudaStream_t)stream);
}

extern "C" int qch_unitarity_defect_c128(const void* d_u, int64_t batch, int64_t n, double* d_defect, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  QCH_CUDA(cudaMemsetAsync(d_defect, 0, sizeof(double) * batch, st));
  int rc = zgemm_defect((const double2*)d_u, d_defect, (int)n, batch, st);
  if (rc) return rc;
  sqrt_kernel<<<(int)((batch + 255) / 256), 256, 0, st>>>(d_defect, batch);
  QCH_LAUNCH_CHECK("sqrt_kernel");
  note_launch(1);
  return QCH_OK;
}
