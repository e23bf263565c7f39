// zgemm.h — complex128 GEMMs on the FP64 tensor pipe (DMMA), shared between
// the translation units of libqcheff (not part of the public C-ABI).
#pragma once
#include <vector>

#include "qch_internal.h"

namespace qch {

enum { ZT_STORE = 0, ZT_ACCUM = 1, ZT_QACC = 2, ZT_UFIN = 3, ZT_DEFECT = 4 };

struct ZtArgs {
  double2* c;           // output (STORE/ACCUM/QACC/UFIN)
  const double2* p[4];  // QACC: P_1..P_nq ; UFIN: p[0] = C (cos part)
  double q[5];          // QACC: q_0..q_nq
  int nq;
  double* acc;  // DEFECT: per-batch sum of squares
  int m, n, k;
  int64_t sc;  // batch stride of C / P (elements; 0 = m n)
  int ldc;     // 0 = n
  // set by the launcher:
  int tn, tm;   // tiles along n, m
  int tiles;    // tiles per matrix
  int nbatch;   // batch items of this launch
  int64_t b0;   // first batch item of this launch
};

// TMA-fed DMMA GEMM (zgemm_tma.cu).  herm: the product is Hermitian (m == n),
// only lower tiles are computed and mirrored.  bh: B is given as Bm (n x k)
// and used as conj(Bm)^T.
int zt_gemm(int mode, bool herm, bool bh, const double2* a, const double2* b, int m, int n, int k, int64_t batch,
            int64_t sa, int64_t sb, ZtArgs g, cudaStream_t st);

// true: 3 real DMMA products per complex product (default), false: 4
bool zgemm_use_3m();
// executed DMMA flops of the TMA kernel since load (accounting)
double dmma_flops_total();

// Hermitian products on the int8 tensor cores (ozgemm.cu: Ozaki slices,
// tcgen05 kind::i8): C = [epilogue] (A B) for Hermitian A, B with A B
// Hermitian; mode ZT_STORE / ZT_QACC (pw, q, nq) / ZT_UFIN (pw[0] = C part)
// Slices are cached per source matrix for the duration of one OzCache (an
// exp(-iH) evaluation reuses Hs, B and B^q on several products); the owner
// drops an entry when it overwrites the matrix.  Component q of an entry:
// 0 Re, 1 Im, 2 Re + Im, 3 Re - Im (slice sets [batch][s][n][n] int8).
struct OzCache {
  struct Entry {
    const void* src = nullptr;
    int8_t* sl[4] = {nullptr, nullptr, nullptr, nullptr};
    int* ex[4] = {nullptr, nullptr, nullptr, nullptr};
  };
  int n;
  int64_t batch;
  cudaStream_t st;
  std::vector<Entry> ent;
  OzCache(int n_, int64_t batch_, cudaStream_t st_) : n(n_), batch(batch_), st(st_) {}
  ~OzCache();
  OzCache(const OzCache&) = delete;
  OzCache& operator=(const OzCache&) = delete;
  int get(const double2* src, unsigned mask, const Entry** out);
  void drop(const void* src);
  void clear();
};
// s_use: leading slices this product uses (0 = all; the expm passes fewer
// for products whose contribution to U is small, see expm_herm)
int zgemm_herm_ozaki(int mode, const double2* a, const double2* b, double2* c, const double2* const* pw,
                     const double* q, int nq, int n, int64_t batch, cudaStream_t st, OzCache* cache = nullptr,
                     int s_use = 0);
bool herm_use_ozaki(int n);
// this thread's next Hermitian products on DMMA regardless of the engine
// (non-finite operands: the int8 slices cannot carry NaN / Inf, DMMA
// propagates them as numpy does)
void herm_force_dmma(bool on);
double oz_int8_ops_total();
int oz_slices();
int herm_engine();  // 1: int8 tensor cores (Ozaki), 0: DMMA

// square / rectangular conveniences (zgemm.cu)
int zgemm(const double2* a, const double2* b, double2* c, int m, int n, int k, int64_t batch, int64_t sa, int64_t sb,
          int64_t sc, cudaStream_t st);
int zgemm_accum(const double2* a, const double2* b, double2* c, int n, int64_t batch, cudaStream_t st);
int zgemm_defect(const double2* u, double* acc, int n, int64_t batch, cudaStream_t st);
// Hermitian products of commuting Hermitian n x n factors (batched)
int zgemm_herm(const double2* a, const double2* b, double2* c, int n, int64_t batch, cudaStream_t st,
               OzCache* oc = nullptr, int s_use = 0);
// C = q0 I + sum_i q_i P_i + A B  (nq <= 4), Hermitian when herm
int zgemm_qacc(bool herm, const double2* a, const double2* b, double2* c, const double2* const* p, const double* q,
               int nq, int n, int64_t batch, cudaStream_t st, OzCache* oc = nullptr, int s_use = 0);
// U = C - i (A B), A B Hermitian
int zgemm_ufin(const double2* a, const double2* b, const double2* cpart, double2* u, int n, int64_t batch,
               cudaStream_t st, OzCache* oc = nullptr, int s_use = 0);

}  // namespace qch
