// capi.cu — error plumbing, device queries and the launch counter of libqcheff.
#include "qch_internal.h"

namespace qch {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int cuda_status(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return QCH_ERR_CUDA;
}
void note_launch(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

int sm_count() {
  int dev = 0, v = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v > 0 ? v : 148;
}
int max_smem_optin() {
  int dev = 0, v = 227 * 1024;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return v;
}

}  // namespace qch

extern "C" int qch_version(void) { return 10000; }

extern "C" size_t qch_last_error(char* buf, size_t len) {
  const std::string& m = qch::g_last_error;
  if (buf && len) {
    size_t k = std::min(len - 1, m.size());
    memcpy(buf, m.data(), k);
    buf[k] = 0;
  }
  return m.size();
}

extern "C" int64_t qch_launch_count(void) { return qch::g_launches.load(); }
