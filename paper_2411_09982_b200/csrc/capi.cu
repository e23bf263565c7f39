// capi.cu — error plumbing, device queries and the launch counter of libqcheff.
#include <map>
#include <mutex>

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
  (void)cudaGetLastError();  // clear the runtime's sticky last-error slot for the next call
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return QCH_ERR_CUDA;
}
void note_launch(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

int sm_count() {
  int dev = 0, v = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v > 0 ? v : 148;
}
// Keep the stream-ordered pool's memory mapped between calls: with the default
// release threshold (0) every synchronising call hands the workspace back to
// the OS and the next cudaMallocAsync re-maps it (hundreds of microseconds).
void ensure_pool() {
  static bool done[64] = {false};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}

cudaError_t smem_attr(const void* func, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  std::lock_guard<std::mutex> lk(mu);
  int& have = done[{func, dev}];
  if (have >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
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

// ---------------------------------------------------------------------------
// In-library kernel timer: CUDA events recorded on the launching stream around
// the hot kernels (npad_run_kernel, magnus_small_k1, zgemm Taylor) while
// enabled; qch_profile_read() synchronises and returns per-name totals.
#include <map>
#include <mutex>
#include <vector>

namespace qch {
struct ProfRec {
  std::string name;
  cudaEvent_t a, b;
};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof_pending;
static std::map<std::string, std::pair<double, long long>> g_prof_acc;

bool prof_on() { return g_prof_on; }
void* prof_begin(const char* name, cudaStream_t st) {
  if (!g_prof_on) return nullptr;
  ProfRec* r = new ProfRec{name, nullptr, nullptr};
  cudaEventCreate(&r->a);
  cudaEventCreate(&r->b);
  cudaEventRecord(r->a, st);
  return r;
}
void prof_end(void* h, cudaStream_t st) {
  if (!h) return;
  ProfRec* r = (ProfRec*)h;
  cudaEventRecord(r->b, st);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_pending.push_back(*r);
  delete r;
}
}  // namespace qch

extern "C" void qch_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(qch::g_prof_mu);
  qch::g_prof_on = on != 0;
}

// Returns the number of names; fills up to cap entries of (total_ms, count)
// and NUL-separated names into names_buf.
extern "C" int qch_profile_read(double* total_ms, int64_t* counts, char* names_buf, int64_t buf_len, int cap,
                                int reset) {
  std::lock_guard<std::mutex> lk(qch::g_prof_mu);
  for (auto& r : qch::g_prof_pending) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    auto& e = qch::g_prof_acc[r.name];
    e.first += ms;
    e.second += 1;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  qch::g_prof_pending.clear();
  int k = 0;
  int64_t off = 0;
  for (auto& kv : qch::g_prof_acc) {
    if (k < cap) {
      total_ms[k] = kv.second.first;
      counts[k] = kv.second.second;
      int64_t L = (int64_t)kv.first.size();
      if (off + L + 1 <= buf_len) {
        memcpy(names_buf + off, kv.first.c_str(), L + 1);
        off += L + 1;
      }
    }
    ++k;
  }
  if (reset) qch::g_prof_acc.clear();
  return k;
}
