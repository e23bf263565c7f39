// qch_internal.h — shared declarations between the CUDA translation units of
// libqcheff (not part of the public C-ABI; see include/qcheff.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <string>

#include "../../include/qcheff.h"

namespace qch {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_status(cudaError_t e, const char* what);

#define QCH_CUDA(call)                                        \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return ::qch::cuda_status(e_, #call); \
  } while (0)

#define QCH_LAUNCH_CHECK(what)                                   \
  do {                                                           \
    cudaError_t e_ = cudaGetLastError();                         \
    if (e_ != cudaSuccess) return ::qch::cuda_status(e_, what); \
  } while (0)

// number of SMs of the current device (cached)
void note_launch(int k);
void* prof_begin(const char* name, cudaStream_t st);
void prof_end(void* h, cudaStream_t st);
int sm_count();
void ensure_pool();
int max_smem_optin();
// raise a kernel's dynamic shared-memory limit on the CURRENT device (the
// attribute is per device; thread-safe, each (kernel, device) set once)
cudaError_t smem_attr(const void* func, int bytes);

}  // namespace qch
