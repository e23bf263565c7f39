// npad_run.h — job/launch interface between the NPAD C-ABI (npad.cu) and the
// persistent greedy drivers (npad_run.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace qch {

struct NpadJob2 {
  double2* h;        // (n, n) matrix, updated in place
  double2* u;        // accumulated unitary (n, n) or nullptr (rows kernel only)
  double* st_q;      // persisted candidate state: keys
  int* st_c;         // partner column (rows kernel) / packed cr (T-rows kernel)
  double2* st_v;     // candidate values
  int* pivots;       // 2*pivot_cap log or nullptr
  long long pivot_cap;
  double threshold;
  long long applied;
  int status;        // 0 converged, 1 max_iter reached, 2 paused at stop_at
  long long stats[4];  // diagnostics: sum(list rows), overflow rotations, short rescans, near-tie fallbacks
};

struct NpadCommon2 {
  int n;
  const unsigned char* inT;  // subspace mask (nullptr = full mode)
  const int* tlist;          // sorted target list
  int n_target;
  int ek;                    // exact keys (q := numpy |z|)
  long long max_iter;
  long long stop_at;
  int stats;                 // 1: accumulate job->stats and printf them at exit
  int* live = nullptr;       // many-chain drivers: chains not yet finished (device counter) ...
  int handover = 0;          // ... pause (status 2) once it is <= handover (the low-latency driver takes over)
};

bool npad_use_trows(const NpadCommon2& cm, bool herm);
int npad_state_init(const double2* h, int64_t batch, const NpadCommon2& cm, bool trows, double* q, int* c,
                    double2* v, cudaStream_t st);
int npad_launch_trows_warp(NpadJob2* jobs, int njobs, const NpadCommon2& cm, cudaStream_t st);
int npad_launch_trows_cta(NpadJob2* jobs, int njobs, const NpadCommon2& cm, cudaStream_t st);
size_t npad_tsmem_bytes(const NpadCommon2& cm);
int npad_launch_tsmem(NpadJob2* jobs, int njobs, const NpadCommon2& cm, cudaStream_t st);
int npad_run_coop(double2* h, int n, double threshold, long long max_iter, int ek, const double* q, const int* c,
                  const double2* v, int* pivots, long long pivot_cap, long long* applied, int* status,
                  cudaStream_t st, double2* u = nullptr);
bool npad_full_warp_ok(const NpadCommon2& cm, bool herm, bool trows);
int npad_launch_full_warp(NpadJob2* jobs, int njobs, const NpadCommon2& cm, cudaStream_t st);
int npad_launch2(NpadJob2* jobs, int njobs, const NpadCommon2& cm, bool herm, bool trows, int pref_threads,
                 bool allow_smem_h, cudaStream_t st);

}  // namespace qch
