// magnus_fused.cu — single-pass Magnus evolve for small N (N <= 4): the
// dim-3 driven transmon of BASELINE config 2.
//
// Reference: evolve() (magnus.py:214-267) = coefficients (:151-169) ->
// effective Hamiltonians (:172-190) -> propagators exp(-i Hbar_n)
// (expm.py:56-71) -> ordered product psi_{n+1} = U_n psi_n (:249-252) with the
// NormDrift check (:270-273).
//
// ONE kernel does all of it in a single pass over the intervals:
//  * a block owns a tile of 128 threads x kR consecutive intervals; each
//    thread forms Hbar_n and U_n in registers (magnus_small.cuh) and the
//    product of its kR propagators;
//  * warp-shuffle inclusive scan of the thread products (3x3 complex, later
//    intervals multiplied on the left), then the 4 warp aggregates;
//  * two-level scan across tiles: a tile publishes its aggregate and arrives
//    at its group (32 consecutive tiles); the group's LAST arrival (warp 0 of
//    its block) scans the group's aggregates, looks back over groups
//    (decoupled look-back, window of 512 groups, nearest published inclusive
//    prefix), and publishes every tile's exclusive prefix E — the other
//    tiles of the group just wait for their flag.  Each tile thus costs one
//    matrix product on the cross-tile critical path instead of a fold over
//    its predecessors;
//  * psi at each thread's start = P_{lane-1} X_warp E psi0; each thread
//    applies its first kR-1 propagators sequentially (the reference's
//    psi <- U psi) and forms its last row as P_lane X_warp E psi0, writing
//    the trajectory rows and checking the norm.
// The ordered product is re-associated (scan), which moves results by
// O(M eps) ~ 1e-12 relative at M = 1e5: inside the 1e-10 parity bar.
//
// Every collective region runs on a provably converged warp (warp index via
// a shuffle, lead condition via a barrier reduction, no divergent code before
// the shuffles): otherwise ptxas guards each shuffle with BRA.DIV and a
// diverged warp takes the serialised WARPSYNC.COLLECTIVE path (measured: 5
// shuffle rounds 3k -> 45k cycles).
//
// A block grabs its next tile right after its prefix arrives (the next
// signal window streams in while the trajectory is written).  Deadlock-free:
// a block waits only for its own group; groups hold at most half the
// resident blocks when tiles outnumber them, so some resident block always
// belongs to a fully grabbed group, and group look-backs wait only on
// earlier groups.
//
// The signals and the trajectory may live in mapped page-locked host memory:
// each tile stages its signal window with one coalesced pass and writes its
// trajectory rows directly, so a host-buffer call streams its I/O over the
// host link while it computes (qch_magnus_evolve_host_c128).
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "magnus_small.cuh"
#include "qch_internal.h"
#include "qch_math.cuh"

namespace qch {

constexpr int kFusedWarps = 4;
constexpr int kFusedThreads = 32 * kFusedWarps;
constexpr int kR = 2;  // consecutive intervals per thread
#ifndef QCH_FUSED_MINB
#define QCH_FUSED_MINB 3  // resident CTAs per SM asked of ptxas for N <= 3 (4: 128 registers + spills, 1.94e9 vs 2.04e9 intervals/s)
#endif
constexpr int kTile = kFusedThreads * kR;  // intervals per tile (one block)

constexpr int kOpsInline = (1 + kMaxK) * 16;

struct FusedArgs {
  SmallArgs s;          // coefficients, operators, order, check, props (s.ubuf, nullable), flags (s.bad)
  const double2* psi0;  // (N,); null: psi0v
  double2 opsv[kOpsInline];  // H0 | H_k by value when s.h0 is null (no upload for the host-buffer call)
  double2 psi0v[4];
  int64_t win;          // > 0: stage each tile's signal window (win samples per control) in shared memory
  int stream_blocks_per_sm;  // > 0: persistent grid of this many blocks per SM streaming the tiles (host I/O)
  const int* chunk_flag;     // non-null: signals arrive in chunks (copy engine); flag = chunks landed
  int tiles_per_chunk;
  // prefix mode (multi-GPU shard, pass 1): no trajectory; store each thread's
  // in-tile exclusive prefix, each tile's exclusive prefix and the block
  // product (s.ubuf receives the propagators)
  double2* pex;        // (M / kR, N, N) or null (full mode)
  double2* etile;      // (tiles, N, N)
  double2* block_out;  // (N, N): U_{M-1} ... U_0
  double2* traj;        // rows (M+1, N), indexed by GLOBAL interval
  int64_t M;            // intervals of the whole evolve
  int64_t tile_begin, tile_end;  // tiles of this launch
  int* tile_ctr;        // this launch's grab counter (zeroed)
  // two-level scan across tiles: groups of 2^gshift consecutive tiles; the
  // last tile of a group to finish scans the group and looks back over groups
  int gshift;
  int* flag;            // per tile: 1 = its exclusive prefix (inc) is ready
  double2* agg;         // per tile N*N: tile aggregate
  double2* inc;         // per tile N*N: tile exclusive prefix
  int* gcount;          // per group: arrivals
  int* gflag;           // per group: 0 none, 1 aggregate, 2 inclusive prefix
  double2* gagg;        // per group N*N
  double2* ginc;        // per group N*N
  // self-cleaning workspace (plan / host-buffer calls): the last block to
  // finish copies the status words to flags_out (nullable) and returns the
  // workspace to its initial state, so a launch needs no memset before it
  int sched_static;               // 1: static round-robin tiles (see the kernel), 0: dynamic grabbing
  int* done_ctr;                  // null: the caller zeroes the workspace per launch
  unsigned long long* flags_out;  // (2,) first non-unitary interval, first norm drift
  unsigned long long* stats;  // non-null (QCH_MAGNUS_STATS): per-block phase cycles, printed by fused_launch
  unsigned long long* tstamp;  // non-null (QCH_MAGNUS_STATS=2): per tile globaltimer at window / prefix / end
};

// phase counters (thread 0 of each block, summed over the block's tiles):
// 0 tiles, 1 wait signals, 2 propagators (thread 0), 3 product + scan + block
// sync, 4 publish + look-back, 5 trajectory + write-out, 6 globaltimer start,
// 7 globaltimer end
constexpr int kStatW = 20;  // + 8 poll cycles, 9 look-back passes, 10 publish cycles, 11 fold cycles
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// acquire/release fence at gpu scope (lighter than __threadfence()'s
// sequentially consistent fence)
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// arrival at a group counter with release semantics (the aggregate stored
// before it is visible to the group's leader): one round trip instead of a
// fence followed by a relaxed atomic
__device__ __forceinline__ int atom_add_release(int* p, int v) {
  int old;
  asm volatile("atom.release.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int W>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(W) : "memory");
}

template <int N>
__device__ __forceinline__ Mat<N> shfl_mat(const Mat<N>& m, int src) {
  Mat<N> o;
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c)
      o.v[r][c] = mkc(__shfl_sync(0xffffffffu, m.v[r][c].re, src), __shfl_sync(0xffffffffu, m.v[r][c].im, src));
  return o;
}
template <int N>
__device__ __forceinline__ Mat<N> shfl_up_mat(const Mat<N>& m, int d) {
  Mat<N> o;
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c)
      o.v[r][c] = mkc(__shfl_up_sync(0xffffffffu, m.v[r][c].re, d), __shfl_up_sync(0xffffffffu, m.v[r][c].im, d));
  return o;
}
template <int N>
__device__ __forceinline__ Mat<N> shfl_down_mat(const Mat<N>& m, int d) {
  Mat<N> o;
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c)
      o.v[r][c] =
          mkc(__shfl_down_sync(0xffffffffu, m.v[r][c].re, d), __shfl_down_sync(0xffffffffu, m.v[r][c].im, d));
  return o;
}
template <int N>
__device__ __forceinline__ void ldcg_mat(Mat<N>& m, const double2* p) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) m.v[r][c] = d2c(__ldcg(p + r * N + c));
}
template <int N>
__device__ __forceinline__ void stcg_mat(double2* p, const Mat<N>& m) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) __stcg(p + r * N + c, c2d(m.v[r][c]));
}

// y = A x
template <int N>
__device__ __forceinline__ void mat_vec(const Mat<N>& a, const cplx* x, cplx* y) {
#pragma unroll
  for (int r = 0; r < N; ++r) {
    double re = 0.0, im = 0.0;
#pragma unroll
    for (int c = 0; c < N; ++c) {
      re = fma(a.v[r][c].re, x[c].re, re);
      re = fma(-a.v[r][c].im, x[c].im, re);
      im = fma(a.v[r][c].re, x[c].im, im);
      im = fma(a.v[r][c].im, x[c].re, im);
    }
    y[r] = mkc(re, im);
  }
}

// ordered product over the lanes of a warp, lane 0 leftmost, of the first
// `span` lanes; the result is broadcast to every lane
template <int N>
__device__ __forceinline__ Mat<N> warp_ordered_product(Mat<N> m, int span, int lane) {
  for (int d = 1; d < span; d <<= 1) {
    const Mat<N> o = shfl_down_mat<N>(m, d);
    if ((lane & (2 * d - 1)) == 0 && lane + d < span) m = mat_mul_fma<N>(m, o);
  }
  return shfl_mat<N>(m, 0);
}

// Exclusive prefix of tile t, E = A_{t-1} ... A_0, by decoupled look-back,
// run by warp 0 alone over a window of up to kLookW predecessors per pass
// (the other warps wait at the next barrier without taking issue slots or
// FP64 pipe cycles — every idle lane of a tree round still costs a full warp
// instruction, so a block-wide look-back in every tile was as expensive as
// forming the propagators):
//  * poll the window's flags (relaxed loads, 16 per lane in flight,
//    __nanosleep back-off) until every predecessor nearer than the nearest
//    published inclusive prefix has published its aggregate; one fence;
//  * lane i folds the L consecutive predecessors at distances [i L, i L + L)
//    (L = ceil(run / 32)), then a 5-round shuffle tree.
// Walks further back only when the window holds no inclusive prefix.
constexpr int kLookK = 16;           // flags per lane
constexpr int kLookW = 32 * kLookK;  // window (predecessors per pass)

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int N>
__device__ Mat<N> warp_lookback(const int* flag, const double2* agg, const double2* inc, int64_t t,
                                unsigned long long* sacc) {
  const int lane = threadIdx.x & 31;
  Mat<N> e = mat_eye<N>();
  int64_t hi = t - 1;  // nearest predecessor not yet folded into e
  while (true) {
    __syncwarp();
    const long long cpoll = sacc != nullptr ? clock64() : 0;
    // distance d = lane + 32 k; predecessor hi - d (< 0: identity prefix)
    unsigned have = 0, incm = 0;  // bit k: aggregate / inclusive published
    int ns = 32, j;
    while (true) {
#pragma unroll
      for (int k = 0; k < kLookK; ++k) {
        if (have & (1u << k)) continue;
        const int64_t p = hi - (lane + 32 * k);
        const int f = p >= 0 ? ld_relaxed(flag + p) : 3;
        if (f != 0) have |= 1u << k;
        if (f >= 2) incm |= 1u << k;
      }
      j = incm ? lane + 32 * (__ffs(incm) - 1) : kLookW;  // nearest inclusive of this lane
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) j = min(j, __shfl_xor_sync(0xffffffffu, j, o));
      const int kneed = (j - lane + 31) / 32;  // k with lane + 32 k < j
      const unsigned need = kneed >= 32 ? 0xffffffffu : ((1u << kneed) - 1u);
      if (__all_sync(0xffffffffu, (have & need) == need)) break;
      __nanosleep(ns);
      ns = min(ns * 2, 256);
    }
    fence_acq_rel();  // acquire side of the flags' release stores
    if (sacc != nullptr && lane == 0) {
      sacc[7] += clock64() - cpoll;
      sacc[8] += 1;
    }
    __syncwarp();
    const int run = min(j + 1, kLookW);  // predecessors folded in this pass
    const int L = (run + 31) / 32;
    Mat<N> m = mat_eye<N>();
    const int d0 = lane * L;
    const int qn = min(L, run - d0);
#pragma unroll 1
    for (int q = 0; q < qn; ++q) {
      const int d = d0 + q;
      const int64_t p = hi - d;
      if (p < 0) break;  // identity prefix
      Mat<N> x;
      ldcg_mat<N>(x, (d < j ? agg : inc) + p * N * N);
      m = q == 0 ? x : mat_mul_fma<N>(m, x);
    }
    __syncwarp();
    e = mat_mul_fma<N>(e, warp_ordered_product<N>(m, (run - 1) / L + 1, lane));
    if (sacc != nullptr && lane == 0) sacc[10] += clock64() - cpoll;
    if (j < kLookW) break;
    hi -= kLookW;
  }
  return e;
}

// The last tile of a group to finish (warp 0 of its block) leads the group:
// scan of the group's tile aggregates (lane i = tile gfirst + i), look-back
// over groups, then every tile's exclusive prefix E = P_{i-1} GE and its flag.
// P_{i-1} and the group aggregate wait in shared scratch (the tile's
// trajectory staging area, free at this point) during the look-back, so the
// look-back's matrices do not push the kernel into local-memory spills.
template <int N>
__device__ __forceinline__ void group_lead(const FusedArgs& g, int64_t gi, int64_t gfirst, int gsize,
                                           double2* scratch, unsigned long long* sacc) {
  const int lane = threadIdx.x & 31;
  // reconverge the warp first: after the divergent publish and the barrier
  // its lanes can still run as separate groups, and every shuffle below would
  // take the compiler's serialised WARPSYNC.COLLECTIVE path (~250 cycles each)
  __syncwarp();
  fence_acq_rel();  // acquire: the group's aggregates
  const long long cl0 = clock64();
  {
    Mat<N> pg = mat_eye<N>();
    if (lane < gsize) ldcg_mat<N>(pg, g.agg + (gfirst + lane) * N * N);
    __syncwarp();
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const Mat<N> q = shfl_up_mat<N>(pg, d);
      if (lane >= d) pg = mat_mul_fma<N>(pg, q);
    }
    Mat<N> px = shfl_up_mat<N>(pg, 1);
    if (lane == 0) px = mat_eye<N>();
    st_mat<N>(scratch + lane * N * N, px);
    if (lane == gsize - 1) {
      st_mat<N>(scratch + 32 * N * N, pg);  // the group aggregate
      if (gi == 0) {
        stcg_mat<N>(g.ginc, pg);
        st_release(g.gflag, 2);
      } else {
        stcg_mat<N>(g.gagg + gi * N * N, pg);
        st_release(g.gflag + gi, 1);
      }
    }
  }
  const long long cl1 = clock64();
  Mat<N> ge = mat_eye<N>();
  if (gi > 0) {
    ge = warp_lookback<N>(g.gflag, g.gagg, g.ginc, gi, sacc);
    __syncwarp();
    if (lane == 0) {
      Mat<N> ga;
      ld_mat<N>(ga, scratch + 32 * N * N);
      stcg_mat<N>(g.ginc + gi * N * N, mat_mul_fma<N>(ga, ge));
      st_release(g.gflag + gi, 2);
    }
  }
  __syncwarp();
  const long long cl2 = clock64();
  if (lane < gsize) {
    Mat<N> px;
    ld_mat<N>(px, scratch + lane * N * N);
    stcg_mat<N>(g.inc + (gfirst + lane) * N * N, mat_mul_fma<N>(px, ge));
    st_release(g.flag + gfirst + lane, 1);
  }
  if (sacc != nullptr && lane == 0) {
    sacc[11] += cl1 - cl0;
    sacc[12] += cl2 - cl1;
    sacc[13] += clock64() - cl2;
    sacc[14] += 1;
  }
}

template <int N>
__global__ void __launch_bounds__(kFusedThreads, (N >= 4 ? 2 : QCH_FUSED_MINB))
    magnus_fused_kernel(const __grid_constant__ FusedArgs g) {
  extern __shared__ __align__(16) double2 fsm[];
  const int K = g.s.ca.K;
  double2* s_ops = fsm;
  const bool inl = g.s.h0 == nullptr;
  load_ops<N>(g.s, s_ops, inl ? g.opsv : nullptr, inl ? g.opsv + N * N : nullptr);
  // warp index through a shuffle (as CUTLASS's canonical_warp_idx_sync): the
  // compiler then knows it is warp-uniform, so shuffles under `warp == 0`
  // compile to plain SHFL instead of the serialised WARPSYNC.COLLECTIVE path
  const int tid = threadIdx.x, lane = tid & 31, warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  double2* s_u = fsm + ops_smem_bytes<N>(K, 2) / sizeof(double2) + (size_t)tid * kR * N * N;
  const size_t wstride = (((size_t)K * g.win + 1) & ~(size_t)1);  // doubles per window buffer (16 B multiple)
  double* s_sig0 = (double*)(fsm + ops_smem_bytes<N>(K, 2) / sizeof(double2) + (size_t)kFusedThreads * kR * N * N);
  // the tile's trajectory rows are staged in the tile's own signal window
  // once the coefficients are formed (the next window prefetches into the
  // other buffer); without staging, or if it is too small, in their own area
  const bool traj_in_window = g.win > 0 && wstride * sizeof(double) >= sizeof(double2) * (size_t)kTile * N;
  double2* s_traj_own = (double2*)(s_sig0 + (g.win > 0 ? 2 * wstride : 0));
  const double2* psi0p = g.psi0 ? g.psi0 : g.psi0v;
  __shared__ Mat<N> s_w[kFusedWarps];    // warp aggregates -> in-block exclusive warp prefixes
  __shared__ Mat<N> s_red[1];            // the tile aggregate
  __shared__ Mat<N> s_e;                 // exclusive prefix of the tile
  __shared__ int s_tile;

  // the control samples of a tile: one coalesced pass into shared memory,
  // issued asynchronously (cp.async) one tile ahead, so that the fetch of the
  // next window — possibly from mapped host memory over the host link —
  // overlaps this tile's arithmetic.  Warps 1-3 issue the host-link traffic
  // (window reads, trajectory writes): warp 0 runs the fenced publish / group
  // protocol, and a fence waits for the issuing thread's own outstanding
  // accesses — an in-flight window read over PCIe cost ~45k cycles per fence
  auto prefetch = [&](int64_t tt, double* buf) {
    const int64_t s0 = tt * kTile * (int64_t)g.s.ca.sub;
    const int64_t cnt = std::min<int64_t>(g.win, g.s.ca.S - s0);
    for (int k = 0; k < K; ++k)
      if (warp > 0)
        for (int64_t q = tid - 32; q < cnt; q += kFusedThreads - 32)
          cp_async8(buf + k * g.win + q, g.s.ca.sig + k * g.s.ca.S + s0 + q);
    cp_commit();
  };

  // signals still streaming in (host-buffer call): wait for the chunk of tile tt
  auto wait_chunk = [&](int64_t tt) {
    if (g.chunk_flag != nullptr && tt < g.tile_end) {
      const int need = (int)(tt / g.tiles_per_chunk) + 1;
      while (ld_acquire(g.chunk_flag) < need) __nanosleep(200);
    }
  };
  __shared__ unsigned long long st_acc[19];  // 6: previous clock, 7 poll, 8 passes, 9 publish
  auto mark = [&](int ph) {
    if (g.stats != nullptr && tid == 0) {
      const unsigned long long c = clock64();
      st_acc[ph] += c - st_acc[6];
      st_acc[6] = c;
    }
  };
  if (g.stats != nullptr && tid == 0) {
    g.stats[blockIdx.x * kStatW + 6] = gtimer();
    for (int q = 0; q < 19; ++q) st_acc[q] = 0;
    st_acc[6] = clock64();
  }
  // tile schedule: static round robin (block b: tiles b, b + grid, ...; the
  // next window is known, so it is prefetched while the current tile is
  // computed — the host-link mode) or dynamic grabbing (load balance)
  const bool stat = g.sched_static != 0;
  if (!stat && tid == 0) {
    s_tile = atomicAdd(g.tile_ctr, 1);
    wait_chunk(g.tile_begin + s_tile);
  }
  __syncthreads();
  int64_t t = stat ? g.tile_begin + blockIdx.x : g.tile_begin + s_tile;
  // the first window; later ones are requested as the previous one lands
  const int64_t G = gridDim.x;
  if (g.win > 0 && t < g.tile_end) prefetch(t, s_sig0);
  for (int it = 0;; ++it) {
    if (t >= g.tile_end) break;
    double* s_sig = s_sig0 + (size_t)(it & 1) * wstride;
    double2* s_traj = traj_in_window ? (double2*)s_sig : s_traj_own;
    const int64_t t_next = t + G;  // static schedule
    if (g.win > 0) cp_wait<0>();
    __syncthreads();
    // static schedule: request the next round's window only now that this
    // one has landed, so the host link serves the windows round by round (in
    // tile order) instead of interleaving every block's rounds
    if (stat && g.win > 0 && t_next < g.tile_end) prefetch(t_next, s_sig0 + (size_t)((it + 1) & 1) * wstride);
    mark(1);
    if (g.stats != nullptr && tid == 0) st_acc[0] += 1;
    if (g.tstamp != nullptr && tid == 0) g.tstamp[t * 4 + 0] = gtimer();
    const int64_t n0 = t * kTile + (int64_t)tid * kR;
    SmallArgs gl = g.s;
    int64_t nbase = 0;
    if (g.win > 0) {
      gl.ca.sig = s_sig;
      gl.ca.S = g.win;
      nbase = t * kTile;
    }

    // ---- propagators of this thread's kR intervals (to shared memory),
    // then their product (registers stay free for the exponential)
#pragma unroll 1
    for (int r = 0; r < kR; ++r) {
      const int64_t n = n0 + r;
      Mat<N> u = mat_eye<N>();
      if (n < g.M) {
        if (g.win > 0 && g.s.ca.sub == 4)
          u = expm_minus_i_fast<N>(interval_hbar_fixed<N, 4>(g.s, s_ops, s_sig, g.win, n - nbase));
        else
          u = expm_minus_i_fast<N>(interval_hbar<N>(gl, s_ops, n - nbase));
        if (g.s.check && !validate_reg<N>(u)) atomicMin(g.s.bad, (unsigned long long)n);
        if (g.s.ubuf != nullptr) st_mat<N>(g.s.ubuf + n * N * N, u);
      }
      st_mat<N>(s_u + r * N * N, u);
    }
    mark(2);
    Mat<N> p;
    ld_mat<N>(p, s_u);
#pragma unroll 1
    for (int r = 1; r < kR; ++r) {
      Mat<N> u;
      ld_mat<N>(u, s_u + r * N * N);
      p = mat_mul_fma<N>(u, p);
    }
    // ---- warp inclusive scan: P_l = A_l ... A_0 (lanes reconverged after the
    // per-lane Taylor degrees, so the shuffles take the converged fast path)
    __syncwarp();
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const Mat<N> q = shfl_up_mat<N>(p, d);
      if (lane >= d) p = mat_mul_fma<N>(p, q);
    }
    if (lane == 31) s_w[warp] = p;
    // P_lane replaces U_{kR-1} in shared memory: the last trajectory row of
    // the thread is P_lane (X_warp E psi0), the earlier ones come from the
    // neighbour's P_{lane-1} and U_0 .. U_{kR-2}; nothing stays in registers
    // across the look-back
    st_mat<N>(s_u + (kR - 1) * N * N, p);
    __syncthreads();
    mark(3);
    // ---- tile aggregate and in-block warp prefixes; arrive at the group
    const int64_t gi = (t - g.tile_begin) >> g.gshift;
    const int64_t gfirst = g.tile_begin + (gi << g.gshift);
    const int gsize = (int)std::min<int64_t>(int64_t(1) << g.gshift, g.tile_end - gfirst);
    // warp 0 forms the tile aggregate (all lanes, same values: no divergent
    // region before the group lead's shuffles), lane 0 publishes it
    bool last = false;
    if (warp == 0) {
      Mat<N> x = s_w[0];
      __syncwarp();
      if (lane == 0) s_w[0] = mat_eye<N>();
#pragma unroll 1
      for (int w = 1; w < kFusedWarps; ++w) {
        const Mat<N> a = s_w[w];
        __syncwarp();
        if (lane == 0) s_w[w] = x;  // exclusive prefix of warp w within the tile
        x = mat_mul_fma<N>(a, x);
      }
      if (lane == 0) {
        s_red[0] = x;  // the tile aggregate
        stcg_mat<N>(g.agg + t * N * N, x);
        last = atom_add_release(g.gcount + gi, 1) == gsize - 1;  // last arrival of the group leads it
      }
      __syncwarp();
    }
    // block-uniform in the compiler's eyes (barrier reduction)
    const bool lead = __syncthreads_or(last);
    if (g.stats != nullptr && tid == 0) st_acc[9] += clock64() - st_acc[6];
    if (warp == 0) {
      if (lead) group_lead<N>(g, gi, gfirst, gsize, s_traj, g.stats != nullptr ? st_acc : nullptr);
      const long long cw0 = clock64();
      if (lane == 0) {
        int ns = 32;
        while (ld_relaxed(g.flag + t) == 0) {
          __nanosleep(ns);
          ns = min(ns * 2, 256);
        }
        fence_acq_rel();  // acquire: the prefix seen flagged
        Mat<N> e;
        ldcg_mat<N>(e, g.inc + t * N * N);
        s_e = e;
        if (g.stats != nullptr) st_acc[15] += clock64() - cw0;
        // dynamic schedule: grab the next tile only now — a block never
        // holds an unstarted tile while it waits for its prefix
        if (!stat) {
          s_tile = atomicAdd(g.tile_ctr, 1);
          wait_chunk(g.tile_begin + s_tile);
        }
      }
    }
    __syncthreads();
    const int64_t tn = stat ? t_next : g.tile_begin + s_tile;
    // dynamic schedule: the next tile's signal window streams in while this
    // tile's trajectory is formed and written
    if (!stat && g.win > 0 && tn < g.tile_end) prefetch(tn, s_sig0 + (size_t)((it + 1) & 1) * wstride);
    mark(4);
    if (g.tstamp != nullptr && tid == 0) g.tstamp[t * 4 + 1] = gtimer();
    if (g.pex != nullptr) {
      // prefix mode: the thread's start = (P_{lane-1} X_warp) E_t psi_start,
      // with psi_start known only after the ranks' exchange
      Mat<N> pexm = mat_eye<N>();
      if (lane > 0) ld_mat<N>(pexm, s_u - kR * N * N + (kR - 1) * N * N);
      st_mat<N>(g.pex + (t * kFusedThreads + tid) * N * N, mat_mul_fma<N>(pexm, s_w[warp]));
      if (tid == 0) {
        st_mat<N>(g.etile + t * N * N, s_e);
        if (t == g.tile_end - 1) st_mat<N>(g.block_out, mat_mul_fma<N>(s_red[0], s_e));
      }
      __syncthreads();  // s_w / s_e reuse
      t = tn;
      continue;
    }
    // ---- trajectory: w = X_warp E psi0; the thread's start state is
    // P_{lane-1} w, its last row P_lane w
    cplx psi0[N], v[N], w[N], x[N];
#pragma unroll
    for (int q = 0; q < N; ++q) psi0[q] = d2c(psi0p[q]);
    mat_vec<N>(s_e, psi0, v);
    mat_vec<N>(s_w[warp], v, w);
    if (lane > 0) {
      Mat<N> pex;
      ld_mat<N>(pex, s_u - kR * N * N + (kR - 1) * N * N);
      mat_vec<N>(pex, w, x);
    } else {
#pragma unroll
      for (int q = 0; q < N; ++q) x[q] = w[q];
    }
    if (t == 0 && tid == 0) {
#pragma unroll
      for (int q = 0; q < N; ++q) g.traj[q] = c2d(psi0[q]);
    }
#pragma unroll 1
    for (int r = 0; r < kR; ++r) {
      const int64_t n = n0 + r;
      if (n >= g.M) break;
      Mat<N> u;
      ld_mat<N>(u, s_u + r * N * N);
      mat_vec<N>(u, r + 1 < kR ? x : w, v);
      double nrm2 = 0.0;
#pragma unroll
      for (int q = 0; q < N; ++q) {
        x[q] = v[q];
        nrm2 = fma(v[q].re, v[q].re, fma(v[q].im, v[q].im, nrm2));
        s_traj[(tid * kR + r) * N + q] = c2d(v[q]);
      }
      if (!(fabs(sqrt(nrm2) - 1.0) <= 1e-6)) atomicMin(g.s.bad + 1, (unsigned long long)n);  // magnus.py:28
    }
    __syncthreads();
    // ---- the tile's trajectory rows leave in one coalesced, contiguous pass
    // (rows t*kTile+1 .. ; the destination may be mapped host memory)
    {
      const int64_t row0 = t * kTile + 1;
      const int64_t rows = std::min<int64_t>(kTile, g.M - t * kTile);
      double2* dst = g.traj + row0 * N;
      if (warp > 0)
        for (int64_t q = tid - 32; q < rows * N; q += kFusedThreads - 32) dst[q] = s_traj[q];
    }
    __syncthreads();  // s_w / s_e / s_traj reuse
    mark(5);
    if (g.tstamp != nullptr && tid == 0) {
      g.tstamp[t * 4 + 2] = gtimer();
      g.tstamp[t * 4 + 3] = blockIdx.x;
    }
    t = tn;
  }
  if (g.done_ctr != nullptr) {
    __shared__ int s_last;
    __syncthreads();
    if (tid == 0) {
      fence_acq_rel();
      s_last = atomicAdd(g.done_ctr, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
      fence_acq_rel();
      const int64_t nt = g.tile_end - g.tile_begin;
      for (int64_t q = tid; q < nt; q += kFusedThreads) {
        g.flag[g.tile_begin + q] = 0;
        g.gflag[q] = 0;
        g.gcount[q] = 0;
      }
      if (tid == 0) {
        if (g.flags_out != nullptr) {
          g.flags_out[0] = g.s.bad[0];
          g.flags_out[1] = g.s.bad[1];
        }
        g.s.bad[0] = ~0ull;
        g.s.bad[1] = ~0ull;
        *g.tile_ctr = 0;
        *g.done_ctr = 0;
      }
    }
  }
  if (g.stats != nullptr && tid == 0) {
#pragma unroll
    for (int q = 0; q < 6; ++q) g.stats[blockIdx.x * kStatW + q] = st_acc[q];
    g.stats[blockIdx.x * kStatW + 7] = gtimer();
    g.stats[blockIdx.x * kStatW + 8] = st_acc[7];
    g.stats[blockIdx.x * kStatW + 9] = st_acc[8];
    g.stats[blockIdx.x * kStatW + 10] = st_acc[9];
    g.stats[blockIdx.x * kStatW + 11] = st_acc[10];
    for (int q = 11; q < 19; ++q) g.stats[blockIdx.x * kStatW + q + 1] = st_acc[q];
  }
}

constexpr size_t kStageMax = 24 * 1024;  // signal window staged in shared memory up to this size (x2 buffers)

template <int N>
static size_t fused_smem(int K) {
  return ops_smem_bytes<N>(K, 2) + sizeof(double2) * (size_t)kFusedThreads * kR * N * N;
}
// samples per control of one tile's window, or 0 when it does not fit
static int64_t fused_window(int K, int sub) {
  const int64_t w = (int64_t)kTile * sub + 1;
  return (K > 0 && (size_t)K * w * sizeof(double) <= kStageMax) ? w : 0;
}

template <int N>
static int fused_launch(FusedArgs& g, cudaStream_t st) {
  g.win = fused_window(g.s.ca.K, g.s.ca.sub);
  const int64_t tiles = g.tile_end - g.tile_begin;
  if (tiles <= 0) return QCH_OK;
  if (const char* e = getenv("QCH_SCHED")) g.sched_static = strcmp(e, "static") == 0 ? 1 : 0;
  if (g.chunk_flag != nullptr) g.sched_static = 0;  // chunked signals: tiles taken in arrival order
  static int smem_optin = 0;
  if (smem_optin == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    int v = 0;
    QCH_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa;
    QCH_CUDA(cudaFuncGetAttributes(&fa, magnus_fused_kernel<N>));
    smem_optin = v - (int)fa.sharedSizeBytes;  // dynamic share of the opt-in maximum
  }
  QCH_CUDA(smem_attr((const void*)magnus_fused_kernel<N>, smem_optin));  // per device
  const size_t wbytes = (((size_t)g.s.ca.K * g.win + 1) & ~(size_t)1) * sizeof(double);
  const size_t tbytes = sizeof(double2) * (size_t)kTile * N;
  const size_t sbase = fused_smem<N>(g.s.ca.K) + (g.win > 0 && wbytes >= tbytes ? 0 : tbytes);
  const size_t smem = sbase + (g.win > 0 ? 2 * wbytes : 0);
  static size_t occ_smem[4] = {0, 0, 0, 0};
  static int occ_val[4] = {0, 0, 0, 0};
  int blocks_per_sm = 0;
  for (int q = 0; q < 4; ++q)
    if (occ_smem[q] == smem) blocks_per_sm = occ_val[q];
  if (blocks_per_sm == 0) {
    QCH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, magnus_fused_kernel<N>, kFusedThreads, smem));
    if (blocks_per_sm < 1) blocks_per_sm = 1;
    static int slot = 0;
    occ_smem[slot & 3] = smem;
    occ_val[slot & 3] = blocks_per_sm;
    ++slot;
  }
  int64_t slots = (int64_t)blocks_per_sm * sm_count();
  if (g.stream_blocks_per_sm > 0) slots = std::min<int64_t>(slots, (int64_t)g.stream_blocks_per_sm * sm_count());
  const int grid = (int)std::min<int64_t>(tiles, slots);
  // group size: 32 tiles, or at most half the resident blocks when the tiles
  // outnumber them (a block waits for its group, so the unfinished top group
  // must never hold every resident block)
  g.gshift = 5;
  if (const char* e = getenv("QCH_GROUP_SHIFT")) g.gshift = std::max(0, std::min(5, atoi(e)));
  if (tiles > grid)  // static schedule: group <= grid suffices; dynamic: <= grid / 2
    while (g.gshift > 0 && (1 << g.gshift) > (g.sched_static ? grid : grid / 2)) --g.gshift;
  static const bool want_stats = getenv("QCH_MAGNUS_STATS") != nullptr;
  static const bool want_ts = want_stats && atoi(getenv("QCH_MAGNUS_STATS")) >= 2;
  static unsigned long long* d_stats = nullptr;
  static unsigned long long* d_ts = nullptr;
  g.stats = nullptr;
  g.tstamp = nullptr;
  if (want_ts && tiles <= 65536) {
    if (d_ts == nullptr) QCH_CUDA(cudaMalloc(&d_ts, sizeof(unsigned long long) * 4 * 65536));
    g.tstamp = d_ts;
  }
  if (want_stats) {
    if (d_stats == nullptr) QCH_CUDA(cudaMalloc(&d_stats, sizeof(unsigned long long) * kStatW * 4096));
    if (grid <= 4096) g.stats = d_stats;
  }
  static const bool trace = getenv("QCH_TRACE") != nullptr;
  const auto tl0 = std::chrono::steady_clock::now();
  void* pr = prof_begin("magnus_fused_kernel", st);
  const auto tl1 = std::chrono::steady_clock::now();
  // Cooperative launch: the tile schedule (static round-robin, or dynamic
  // with group waits) needs every block of the grid resident at once; a
  // cooperative launch guarantees that (or fails cleanly) even when other
  // kernels share the GPU.
  // QCH_FUSED_COOP: 1 always, 0 never, 2 (default) for the static schedule
  // only — there every block owns fixed tiles, so a non-resident block would
  // stall the scan; the dynamic schedule hands tiles only to running blocks
  // and keeps every group within half the grid
  static const int coop_mode = getenv("QCH_FUSED_COOP") ? atoi(getenv("QCH_FUSED_COOP")) : 2;
  if (coop_mode == 1 || (coop_mode == 2 && g.sched_static)) {
    void* kargs[] = {(void*)&g};
    QCH_CUDA(cudaLaunchCooperativeKernel((const void*)magnus_fused_kernel<N>, dim3(grid), dim3(kFusedThreads), kargs,
                                         smem, st));
  } else {
    magnus_fused_kernel<N><<<grid, kFusedThreads, smem, st>>>(g);
  }
  const auto tl2 = std::chrono::steady_clock::now();
  prof_end(pr, st);
  if (trace)
    fprintf(stderr, "[qch trace] fused launch: prof %.1f us, <<<>>> %.1f us (params %zu B, grid %d, smem %zu)\n",
            std::chrono::duration<double, std::micro>(tl1 - tl0).count(),
            std::chrono::duration<double, std::micro>(tl2 - tl1).count(), sizeof(g), grid, smem);
  QCH_LAUNCH_CHECK("magnus_fused_kernel");
  if (g.stats != nullptr) {
    std::vector<unsigned long long> h((size_t)kStatW * grid);
    QCH_CUDA(cudaMemcpyAsync(h.data(), d_stats, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    QCH_CUDA(cudaStreamSynchronize(st));
    double sum[6] = {0, 0, 0, 0, 0, 0}, mx[6] = {0, 0, 0, 0, 0, 0};
    unsigned long long t0 = ~0ull, t1 = 0, s_last = 0, e_first = ~0ull;
    for (int b = 0; b < grid; ++b) {
      for (int q = 0; q < 6; ++q) {
        sum[q] += (double)h[b * kStatW + q];
        mx[q] = std::max(mx[q], (double)h[b * kStatW + q]);
      }
      t0 = std::min(t0, h[b * kStatW + 6]);
      s_last = std::max(s_last, h[b * kStatW + 6]);
      e_first = std::min(e_first, h[b * kStatW + 7]);
      t1 = std::max(t1, h[b * kStatW + 7]);
    }
    double ext[4] = {0, 0, 0, 0};
    for (int b = 0; b < grid; ++b)
      for (int q = 0; q < 4; ++q) ext[q] += (double)h[b * kStatW + 8 + q];
    const double tiles = sum[0] > 0 ? sum[0] : 1;
    fprintf(stderr,
            "[qch magnus stats] look-back per tile: publish %.0f cycles, poll %.0f cycles, poll+fold %.0f cycles, "
            "passes %.2f\n",
            ext[2] / tiles, ext[0] / tiles, ext[3] / tiles, ext[1] / tiles);
    double ld[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int b = 0; b < grid; ++b)
      for (int q = 0; q < 8; ++q) ld[q] += (double)h[b * kStatW + 12 + q];
    const double nl = ld[3] > 0 ? ld[3] : 1;
    if (g.tstamp != nullptr) {  // per-tile timeline for tools/tstamp_view.py
      std::vector<unsigned long long> ts((size_t)4 * tiles);
      QCH_CUDA(cudaMemcpy(ts.data(), d_ts, ts.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
      if (FILE* f = fopen("gpurun_out/magnus_tstamp.csv", "w")) {
        fprintf(f, "tile,block,window_ns,prefix_ns,end_ns\n");
        for (int64_t q = 0; q < tiles; ++q)
          fprintf(f, "%lld,%llu,%lld,%lld,%lld\n", (long long)q, ts[q * 4 + 3], (long long)(ts[q * 4] - t0),
                  (long long)(ts[q * 4 + 1] - t0), (long long)(ts[q * 4 + 2] - t0));
        fclose(f);
      }
    }
    fprintf(stderr,
            "[qch magnus stats] group leaders %.0f: scan %.0f, look-back %.0f, prefixes %.0f cycles; tile wait for "
            "prefix %.0f cycles\n",
            ld[3], ld[0] / nl, ld[1] / nl, ld[2] / nl, ld[4] / tiles);
    fprintf(stderr,
            "[qch magnus stats] grid %d smem %zu tiles %.0f | cycles/tile: wait %.0f (max %.0f) prop %.0f (max %.0f) "
            "scan %.0f (max %.0f) lookback %.0f (max %.0f) traj %.0f (max %.0f) | block start spread %.2f us, "
            "first end %.2f us, last end %.2f us\n",
            grid, smem, sum[0], sum[1] / tiles, mx[1], sum[2] / tiles, mx[2], sum[3] / tiles, mx[3], sum[4] / tiles,
            mx[4], sum[5] / tiles, mx[5], (s_last - t0) * 1e-3, (e_first - t0) * 1e-3, (t1 - t0) * 1e-3);
  }
  note_launch(1);
  return QCH_OK;
}

int fused_launch_any(int n, FusedArgs& g, cudaStream_t st) {
  switch (n) {
    case 1: return fused_launch<1>(g, st);
    case 2: return fused_launch<2>(g, st);
    case 3: return fused_launch<3>(g, st);
    default: return fused_launch<4>(g, st);
  }
}

int64_t fused_tiles(int64_t M) { return (M + kTile - 1) / kTile; }
int64_t fused_tile_intervals() { return kTile; }

// workspace: [tile flags | counters | group flags | group arrivals | done]
// (zeroed) | bad (2 ull, all ones) | agg | inc | gagg | ginc
size_t fused_ws_bytes(int64_t N, int64_t M, int nlaunch) {
  const int64_t nt = fused_tiles(M);
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  return al(sizeof(int) * (3 * nt + nlaunch + 1)) + al(16) + 4 * al(sizeof(double2) * N * N * nt);
}
size_t fused_ws_zero_bytes(int64_t M, int nlaunch) {
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  return al(sizeof(int) * (3 * fused_tiles(M) + nlaunch + 1));
}
void fused_carve(void* ws, int64_t N, int64_t M, int nlaunch, FusedArgs* g, int** ctr) {
  const int64_t nt = fused_tiles(M);
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  unsigned char* p = (unsigned char*)ws;
  g->flag = (int*)p;
  *ctr = g->flag + nt;
  g->gflag = *ctr + nlaunch;
  g->gcount = g->gflag + nt;
  g->sched_static = 1;  // static round-robin tiles, cooperative launch (measured faster than dynamic grabbing)
  g->tstamp = nullptr;
  g->done_ctr = nullptr;  // set by the self-cleaning callers
  g->flags_out = nullptr;
  p += al(sizeof(int) * (3 * nt + nlaunch + 1));
  g->s.bad = (unsigned long long*)p;
  p += al(16);
  const size_t mb = al(sizeof(double2) * N * N * nt);
  g->agg = (double2*)p;
  g->inc = (double2*)(p + mb);
  g->gagg = (double2*)(p + 2 * mb);
  g->ginc = (double2*)(p + 3 * mb);
}

namespace {
struct Trace {
  bool on = getenv("QCH_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[qch trace] %-28s %8.1f us\n", what, std::chrono::duration<double, std::micro>(t - t0).count());
  }
};
struct FBuf {
  cudaStream_t st;
  void* p = nullptr;
  explicit FBuf(cudaStream_t s) : st(s) {}
  cudaError_t alloc(size_t b) {
    ensure_pool();
    return cudaMallocAsync(&p, std::max<size_t>(b, 16), st);
  }
  ~FBuf() {
    if (p) cudaFreeAsync(p, st);
  }
};

// page-locked status words of the host-buffer call (one pair per device)
struct Pipe {
  std::mutex mu;  // one host-buffer call at a time per device (shared workspace + status words)
  unsigned long long* h_flags = nullptr;
  cudaStream_t in = nullptr;  // copy stream of the host-buffer call
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int* d_flag = nullptr;      // chunk counter (cudaMalloc: stream memory ops reject pool memory)
  void* ws = nullptr;         // self-cleaning fused workspace of the host-buffer call
  size_t ws_bytes = 0;
  int64_t ws_n = 0, ws_m = 0;
  bool ws_dirty = true;
};
Pipe& pipe_for_device() {
  static Pipe pipes[64];
  int dev = 0;
  cudaGetDevice(&dev);
  Pipe& p = pipes[dev & 63];
  static std::mutex init_mu;
  std::lock_guard<std::mutex> lk(init_mu);
  if (p.h_flags == nullptr) {
    cudaHostAlloc(&p.h_flags, 2 * sizeof(unsigned long long), cudaHostAllocMapped);
    cudaStreamCreateWithFlags(&p.in, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&p.ev0, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&p.ev1, cudaEventDisableTiming);
    cudaMalloc(&p.d_flag, 256);
  }
  return p;
}

// cuStreamWriteValue32 (driver API, fetched through the runtime): a copy
// stream bumps a device flag after each chunk it lands, and the running
// kernel polls it
typedef int (*WriteValue32Fn)(cudaStream_t, unsigned long long, unsigned, unsigned);
WriteValue32Fn write_value32() {
  static WriteValue32Fn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &p, 12000, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (WriteValue32Fn)p;
    else
      cudaGetLastError();
  }
  return fn;
}

// device address of a page-locked, mapped host buffer (UVA), or null for
// pageable memory
void* mapped_ptr(const void* h) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return (a.type == cudaMemoryTypeHost) ? a.devicePointer : nullptr;
}
}  // namespace

// Initial state of a self-cleaning workspace (zero counters, all-ones status
// words); the kernel's last block restores it after every launch.
int fused_ws_init(void* ws, int64_t N, int64_t M, cudaStream_t st) {
  FusedArgs g;
  int* ctr = nullptr;
  fused_carve(ws, N, M, 1, &g, &ctr);
  QCH_CUDA(cudaMemsetAsync(ws, 0, fused_ws_zero_bytes(M, 1), st));
  QCH_CUDA(cudaMemsetAsync(g.s.bad, 0xff, 2 * sizeof(unsigned long long), st));
  return QCH_OK;
}
static int* fused_done_ptr(const FusedArgs& g, int64_t M) { return g.gcount + fused_tiles(M); }

// Device-buffer fused evolve (N <= 4).  d_flags_out non-null: copy the two
// status words there and return without synchronising (async evolve).
// d_work non-null: a self-cleaning workspace (fused_ws_init) — the launch is
// then the only operation (no allocation, memset or copy around it).
int fused_evolve_device(const SmallArgs& base, int64_t N, int64_t M, const double2* d_psi0, double2* d_traj,
                        int64_t* bad_index, unsigned long long* d_flags_out, cudaStream_t st, void* d_work) {
  FBuf ws(st);
  if (d_work == nullptr) QCH_CUDA(ws.alloc(fused_ws_bytes(N, M, 1)));
  FusedArgs g;
  g.s = base;
  g.stream_blocks_per_sm = 0;
  g.chunk_flag = nullptr;
  g.tiles_per_chunk = 1;
  g.pex = nullptr;
  g.etile = nullptr;
  g.block_out = nullptr;
  int* ctr = nullptr;
  fused_carve(d_work ? d_work : ws.p, N, M, 1, &g, &ctr);
  if (d_work != nullptr) {
    g.done_ctr = fused_done_ptr(g, M);
    g.flags_out = d_flags_out;
  } else {
    QCH_CUDA(cudaMemsetAsync(ws.p, 0, fused_ws_zero_bytes(M, 1), st));
    QCH_CUDA(cudaMemsetAsync(g.s.bad, 0xff, 2 * sizeof(unsigned long long), st));
  }
  g.psi0 = d_psi0;
  g.traj = d_traj;
  g.M = M;
  g.tile_begin = 0;
  g.tile_end = fused_tiles(M);
  g.tile_ctr = ctr;
  if (int rc = fused_launch_any((int)N, g, st)) return rc;
  if (d_work != nullptr) {
    if (d_flags_out) return QCH_OK;
    return fail(QCH_ERR_VALUE, "a self-cleaning workspace needs a flags buffer");
  }
  if (d_flags_out) {
    QCH_CUDA(cudaMemcpyAsync(d_flags_out, g.s.bad, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, st));
    return QCH_OK;
  }
  unsigned long long b[2];
  QCH_CUDA(cudaMemcpyAsync(b, g.s.bad, sizeof b, cudaMemcpyDeviceToHost, st));
  QCH_CUDA(cudaStreamSynchronize(st));
  if (base.check && b[0] != ~0ull) {
    if (bad_index) *bad_index = (int64_t)b[0];
    return fail(QCH_ERR_NONFINITE, "propagator not unitary (interval " + std::to_string(b[0]) + ")");
  }
  if (b[1] != ~0ull) {
    if (bad_index) *bad_index = (int64_t)b[1];
    return fail(QCH_ERR_NORM_DRIFT, "state norm drifted after interval " + std::to_string(b[1]));
  }
  return QCH_OK;
}

}  // namespace qch


namespace qch {
// ---------------------------------------------------------------------------
// Multi-GPU interval sharding, N <= 4.  Pass 1 (prepare):
// the fused kernel in prefix mode — propagators, in-tile and tile prefixes,
// the rank's block product B_r.  The ranks all-gather the B's.  Pass 2
// (finish): psi_start = B_{r-1}...B_0 psi0 (qch_magnus_apply_prefix_c128),
// then every thread's start state is one mat-vec chain from the stored
// prefixes and its 2 propagators give its trajectory rows.
template <int N>
__global__ void __launch_bounds__(128) shard_traj_kernel(const double2* __restrict__ ustash,
                                                         const double2* __restrict__ pex,
                                                         const double2* __restrict__ etile,
                                                         const double2* __restrict__ psi_start, int64_t M,
                                                         double2* __restrict__ traj, unsigned long long* bad) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // thread slot of pass 1
  const int64_t n0 = k * kR;
  cplx ps[N], v[N], w[N];
#pragma unroll
  for (int q = 0; q < N; ++q) ps[q] = d2c(psi_start[q]);
  if (k == 0) {
#pragma unroll
    for (int q = 0; q < N; ++q) traj[q] = c2d(ps[q]);
  }
  if (n0 >= M) return;
  Mat<N> e, pm;
  ld_mat<N>(e, etile + (k / kFusedThreads) * N * N);
  ld_mat<N>(pm, pex + k * N * N);
  mat_vec<N>(e, ps, v);
  mat_vec<N>(pm, v, w);
#pragma unroll 1
  for (int r = 0; r < kR; ++r) {
    const int64_t n = n0 + r;
    if (n >= M) break;
    Mat<N> u;
    ld_mat<N>(u, ustash + n * N * N);
    mat_vec<N>(u, w, v);
    double nrm2 = 0.0;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      w[q] = v[q];
      nrm2 = fma(v[q].re, v[q].re, fma(v[q].im, v[q].im, nrm2));
      traj[(n + 1) * N + q] = c2d(v[q]);
    }
    if (!(fabs(sqrt(nrm2) - 1.0) <= 1e-6)) atomicMin(bad + 1, (unsigned long long)n);  // magnus.py:28
  }
}

// workspace: fused state | U (M) | thread prefixes (tiles * 128) | tile prefixes (tiles)
size_t shard_ws_bytes(int64_t N, int64_t M) {
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const int64_t tiles = fused_tiles(M);
  return al(fused_ws_bytes(N, M, 1)) + al(sizeof(double2) * N * N * M) +
         al(sizeof(double2) * N * N * tiles * kFusedThreads) + al(sizeof(double2) * N * N * tiles);
}
struct ShardWs {
  unsigned char* fused;
  double2* u;
  double2* pex;
  double2* etile;
};
ShardWs shard_carve(void* ws, int64_t N, int64_t M) {
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const int64_t tiles = fused_tiles(M);
  ShardWs w;
  w.fused = (unsigned char*)ws;
  w.u = (double2*)(w.fused + al(fused_ws_bytes(N, M, 1)));
  w.pex = (double2*)((unsigned char*)w.u + al(sizeof(double2) * N * N * M));
  w.etile = (double2*)((unsigned char*)w.pex + al(sizeof(double2) * N * N * tiles * kFusedThreads));
  return w;
}

int shard_prepare(const SmallArgs& base, int64_t N, int64_t M, void* d_work, double2* d_block, cudaStream_t st) {
  ShardWs w = shard_carve(d_work, N, M);
  FusedArgs g;
  g.s = base;
  g.s.ubuf = w.u;
  int* ctr = nullptr;
  fused_carve(w.fused, N, M, 1, &g, &ctr);
  QCH_CUDA(cudaMemsetAsync(w.fused, 0, fused_ws_zero_bytes(M, 1), st));
  QCH_CUDA(cudaMemsetAsync(g.s.bad, 0xff, 2 * sizeof(unsigned long long), st));
  g.psi0 = nullptr;
  g.traj = nullptr;
  g.M = M;
  g.tile_begin = 0;
  g.tile_end = fused_tiles(M);
  g.tile_ctr = ctr;
  g.stream_blocks_per_sm = 0;
  g.chunk_flag = nullptr;
  g.tiles_per_chunk = 1;
  g.pex = w.pex;
  g.etile = w.etile;
  g.block_out = d_block;
  return fused_launch_any((int)N, g, st);
}

int shard_finish(int64_t N, int64_t M, void* d_work, const double2* d_psi_start, double2* d_traj,
                 unsigned long long** bad_out, cudaStream_t st) {
  ShardWs w = shard_carve(d_work, N, M);
  FusedArgs g;
  int* ctr = nullptr;
  fused_carve(w.fused, N, M, 1, &g, &ctr);
  const int64_t threads = fused_tiles(M) * kFusedThreads;
  const unsigned blocks = (unsigned)((threads + 127) / 128);
  void* pr = prof_begin("shard_traj_kernel", st);
  switch (N) {
    case 1: shard_traj_kernel<1><<<blocks, 128, 0, st>>>(w.u, w.pex, w.etile, d_psi_start, M, d_traj, g.s.bad); break;
    case 2: shard_traj_kernel<2><<<blocks, 128, 0, st>>>(w.u, w.pex, w.etile, d_psi_start, M, d_traj, g.s.bad); break;
    case 3: shard_traj_kernel<3><<<blocks, 128, 0, st>>>(w.u, w.pex, w.etile, d_psi_start, M, d_traj, g.s.bad); break;
    default: shard_traj_kernel<4><<<blocks, 128, 0, st>>>(w.u, w.pex, w.etile, d_psi_start, M, d_traj, g.s.bad); break;
  }
  prof_end(pr, st);
  QCH_LAUNCH_CHECK("shard_traj_kernel");
  note_launch(1);
  *bad_out = g.s.bad;
  return QCH_OK;
}

}  // namespace qch

using namespace qch;

extern "C" int qch_magnus_evolve_c128(const void* d_h0, const void* d_hk, const void* d_comm, int64_t K, int64_t N,
                                      const double* d_sig, int64_t S, double t_start, double t_end, int64_t M,
                                      int order, const void* d_psi0, void* d_traj, void* d_props, int check,
                                      int64_t* bad_index, void* stream);

// evolve() with HOST buffers (magnus.py:214-267): inputs are read from and the
// trajectory written to host memory.  For N <= 4 one fused launch streams the
// page-locked buffers over the host link itself (zero-copy), so transfers and
// compute overlap; pageable buffers are staged through device memory.
// np.linspace(t0, t1, n) bit for bit (numpy/_core/function_base.py):
// step = (t1 - t0) / (n - 1); y_i = i * step + t0 (two roundings, no FMA);
// a zero (underflowed) step takes numpy's (i / div) * delta branch; the last
// point is t1 exactly.
static void np_linspace(double t0, double t1, int64_t n, double* y) {
  if (n <= 0) return;
  const int64_t div = n - 1;
  volatile double delta = t1 - t0;
  if (div > 0) {
    const double step = delta / (double)div;
    if (step == 0.0) {
      for (int64_t i = 0; i < n; ++i) {
        volatile double q = (double)i / (double)div;
        volatile double r = q * delta;
        y[i] = r + t0;
      }
    } else {
      for (int64_t i = 0; i < n; ++i) {
        volatile double r = (double)i * step;
        y[i] = r + t0;
      }
    }
    y[n - 1] = t1;
  } else {
    volatile double r = 0.0 * delta;
    y[0] = r + t0;
  }
}

extern "C" int qch_magnus_evolve_host_c128(const void* h_h0, const void* h_hk, int64_t K, int64_t N,
                                           const double* h_sig, int64_t S, double t_start, double t_end, int64_t M,
                                           int order, const void* h_psi0, void* h_traj, int check,
                                           int64_t* bad_index, double* h_times, void* stream) {
  if (M < 1) return fail(QCH_ERR_GRID, "need at least one interval");
  if ((S - 1) % M)
    return fail(QCH_ERR_GRID, std::to_string(M) + " intervals do not divide " + std::to_string(S - 1) + " sample steps");
  if (order != 1 && order != 2) return fail(QCH_ERR_VALUE, "order must be 1 or 2");
  if (N < 1) return fail(QCH_ERR_VALUE, "dimension must be at least 1");
  cudaStream_t st = (cudaStream_t)stream;
  Trace tr;
  const int64_t nn = N * N;
  const int64_t Kd = std::max<int64_t>(K, 1);
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };

  if (N > 4 || K > kMaxK) {  // generic path: upload, device evolve, download
    FBuf dev(st);
    const size_t b_ops = al(sizeof(double2) * nn * (1 + Kd)), b_psi = al(sizeof(double2) * N),
                 b_sig = al(sizeof(double) * Kd * S), b_traj = al(sizeof(double2) * N * (M + 1));
    QCH_CUDA(dev.alloc(b_ops + b_psi + b_sig + b_traj));
    unsigned char* base = (unsigned char*)dev.p;
    double2* d_h0 = (double2*)base;
    double2* d_hk = d_h0 + nn;
    double2* d_psi0 = (double2*)(base + b_ops);
    double* d_sig = (double*)(base + b_ops + b_psi);
    double2* d_traj = (double2*)(base + b_ops + b_psi + b_sig);
    QCH_CUDA(cudaMemcpyAsync(d_h0, h_h0, sizeof(double2) * nn, cudaMemcpyHostToDevice, st));
    if (K > 0) QCH_CUDA(cudaMemcpyAsync(d_hk, h_hk, sizeof(double2) * nn * K, cudaMemcpyHostToDevice, st));
    QCH_CUDA(cudaMemcpyAsync(d_psi0, h_psi0, sizeof(double2) * N, cudaMemcpyHostToDevice, st));
    if (K > 0) QCH_CUDA(cudaMemcpyAsync(d_sig, h_sig, sizeof(double) * K * S, cudaMemcpyHostToDevice, st));
    else QCH_CUDA(cudaMemsetAsync(d_sig, 0, sizeof(double) * S, st));
    if (int rc = qch_magnus_evolve_c128(d_h0, d_hk, nullptr, K, N, d_sig, S, t_start, t_end, M, order, d_psi0,
                                        d_traj, nullptr, check, bad_index, stream))
      return rc;
    QCH_CUDA(cudaMemcpyAsync(h_traj, d_traj, sizeof(double2) * N * (M + 1), cudaMemcpyDeviceToHost, st));
    if (h_times) np_linspace(t_start, t_end, M + 1, h_times);
    QCH_CUDA(cudaStreamSynchronize(st));
    return QCH_OK;
  }

  // N <= 4: ONE allocation, two memsets, ONE launch.  Operators and psi0
  // travel inside the kernel arguments; page-locked (mapped) signal /
  // trajectory buffers are read and written by the kernel directly over the
  // host link, so the H2D of the signals, the compute and the D2H of the
  // trajectory all overlap.
  // signals: page-locked -> read zero-copy by the kernel (measured fastest
  // end to end); pageable -> one staged copy before the kernel.
  // QCH_SIG_MODE=copy|stream selects a copy-engine H2D instead (stream: in
  // chunks, each bumping a flag the running kernel polls).
  const char* smode = getenv("QCH_SIG_MODE");
  const bool pinned_sig = K > 0 && mapped_ptr(h_sig) != nullptr;
  const bool sig_stream = pinned_sig && smode != nullptr && strcmp(smode, "stream") == 0 && write_value32() != nullptr;
  const bool sig_map = pinned_sig && !sig_stream && !(smode != nullptr && strcmp(smode, "copy") == 0);
  const double* sig = sig_map ? (const double*)mapped_ptr(h_sig) : nullptr;
  double2* traj = getenv("QCH_NOMAP_TRAJ") ? nullptr : (double2*)mapped_ptr(h_traj);
  const size_t b_sig = sig ? 0 : al(sizeof(double) * Kd * S);
  const size_t b_traj = traj ? 0 : al(sizeof(double2) * N * (M + 1));
  FBuf dev(st);
  if (b_sig + b_traj > 0) QCH_CUDA(dev.alloc(b_sig + b_traj));
  double* d_sig = (double*)dev.p;
  double2* d_traj = (double2*)((unsigned char*)dev.p + b_sig);
  if (sig == nullptr) {
    if (K > 0 && !sig_stream) QCH_CUDA(cudaMemcpyAsync(d_sig, h_sig, sizeof(double) * K * S, cudaMemcpyHostToDevice, st));
    sig = d_sig;
  }
  if (traj == nullptr) traj = d_traj;
  Pipe& pp = pipe_for_device();
  // the device's self-cleaning workspace (grown on demand) and status words:
  // concurrent callers on one device (ctypes releases the GIL) take turns
  std::lock_guard<std::mutex> call_lock(pp.mu);
  const size_t b_ws = fused_ws_bytes(N, M, 1);
  if (pp.ws_bytes < b_ws || pp.ws_dirty || pp.ws_n != N || pp.ws_m != M) {  // the layout depends on (N, M)
    if (pp.ws != nullptr && pp.ws_bytes < b_ws) {
      QCH_CUDA(cudaFree(pp.ws));
      pp.ws = nullptr;
    }
    if (pp.ws == nullptr) {
      QCH_CUDA(cudaMalloc(&pp.ws, b_ws));
      pp.ws_bytes = b_ws;
    }
    pp.ws_dirty = true;  // until the initialisation below is known to have run
    pp.ws_n = N;
    pp.ws_m = M;
  }
  tr.mark("buffers");
  const int64_t sub = (S - 1) / M;
  FusedArgs g;
  memcpy(g.opsv, h_h0, sizeof(double2) * nn);
  if (K > 0) memcpy(g.opsv + nn, h_hk, sizeof(double2) * nn * K);
  memcpy(g.psi0v, h_psi0, sizeof(double2) * N);
  // host-link I/O: a persistent grid streams the tiles so fetches, arithmetic
  // and write-backs of different tiles overlap
  g.stream_blocks_per_sm = (sig != d_sig || traj != d_traj) ? 1 : 0;  // zero-copy I/O: persistent grid
  if (const char* e = getenv("QCH_STREAM_BPS")) g.stream_blocks_per_sm = atoi(e);

  int* ctr = nullptr;
  fused_carve(pp.ws, N, M, 1, &g, &ctr);
  if (pp.ws_dirty)
    if (int rc = fused_ws_init(pp.ws, N, M, st)) return rc;
  g.done_ctr = fused_done_ptr(g, M);
  tr.mark("workspace");
  g.flags_out = (unsigned long long*)mapped_ptr(pp.h_flags);  // status words straight into page-locked memory
  tr.mark("flags ptr");
  // host-link I/O: static tile schedule, so each block prefetches its next
  // signal window while it computes the current tile
  g.sched_static = g.stream_blocks_per_sm > 0 ? 1 : 0;
  g.s.ca = CoefArgs{sig, (int)K, S, M, (int)sub, (t_end - t_start) / (double)(S - 1)};
  g.s.h0 = nullptr;  // operators inline (g.opsv)
  g.s.hk = nullptr;
  g.s.comm = nullptr;  // formed in the kernel preamble
  g.s.order = order;
  g.s.dt_int = (t_end - t_start) / (double)M;
  g.s.check = check;
  g.s.ubuf = nullptr;
  g.psi0 = nullptr;
  g.traj = traj;
  g.M = M;
  g.tile_begin = 0;
  g.tile_end = fused_tiles(M);
  g.tile_ctr = ctr;
  g.chunk_flag = nullptr;
  g.tiles_per_chunk = 1;
  g.pex = nullptr;
  g.etile = nullptr;
  g.block_out = nullptr;
  if (sig_stream) {
    const int64_t tiles = fused_tiles(M);
    int nch = (int)std::min<int64_t>(8, tiles);
    if (const char* e = getenv("QCH_SIG_CHUNKS")) nch = std::max(1, std::min((int)tiles, atoi(e)));
    const int tpc = (int)((tiles + nch - 1) / nch);
    nch = (int)((tiles + tpc - 1) / tpc);
    int* d_flag = pp.d_flag;
    QCH_CUDA(cudaMemsetAsync(d_flag, 0, sizeof(int), st));
    QCH_CUDA(cudaEventRecord(pp.ev0, st));  // flag reset + buffers ready before the copies
    QCH_CUDA(cudaStreamWaitEvent(pp.in, pp.ev0, 0));
    for (int c = 0; c < nch; ++c) {
      const int64_t s0 = (int64_t)c * tpc * fused_tile_intervals() * sub;
      const int64_t s1 = std::min<int64_t>(S, (int64_t)(c + 1) * tpc * fused_tile_intervals() * sub + 1);
      QCH_CUDA(cudaMemcpy2DAsync(d_sig + s0, sizeof(double) * S, h_sig + s0, sizeof(double) * S,
                                 sizeof(double) * (s1 - s0), K, cudaMemcpyHostToDevice, pp.in));
      const int wr = write_value32()(pp.in, (unsigned long long)(uintptr_t)d_flag, (unsigned)(c + 1), 0);
      if (wr != 0) return fail(QCH_ERR_CUDA, "cuStreamWriteValue32 failed: CUresult " + std::to_string(wr));
    }
    QCH_CUDA(cudaEventRecord(pp.ev1, pp.in));
    g.chunk_flag = d_flag;
    g.tiles_per_chunk = tpc;
    g.stream_blocks_per_sm = 0;
  }
  tr.mark("args");
  if (int rc = fused_launch_any((int)N, g, st)) return rc;
  tr.mark("launched");
  if (sig_stream) QCH_CUDA(cudaStreamWaitEvent(st, pp.ev1, 0));  // copies retired before the buffers are freed
  if (traj == d_traj)
    QCH_CUDA(cudaMemcpyAsync(h_traj, d_traj, sizeof(double2) * N * (M + 1), cudaMemcpyDeviceToHost, st));
  tr.mark("enqueued");
  if (h_times) np_linspace(t_start, t_end, M + 1, h_times);  // on the host while the kernel runs
  tr.mark("times");
  QCH_CUDA(cudaStreamSynchronize(st));
  pp.ws_dirty = false;  // the kernel ran to completion: workspace clean again
  tr.mark("synchronized");
  const unsigned long long b0 = pp.h_flags[0], b1 = pp.h_flags[1];
  if (check && b0 != ~0ull) {
    if (bad_index) *bad_index = (int64_t)b0;
    return fail(QCH_ERR_NONFINITE, "propagator not unitary (interval " + std::to_string(b0) + ")");
  }
  if (b1 != ~0ull) {
    if (bad_index) *bad_index = (int64_t)b1;
    return fail(QCH_ERR_NORM_DRIFT, "state norm drifted after interval " + std::to_string(b1));
  }
  return QCH_OK;
}
