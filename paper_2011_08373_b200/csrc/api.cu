// api.cu -- error plumbing, version, workspace query, launch accounting and
// CUDA-event profiling of libgrsolve.
#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

static thread_local std::string g_err;

void gr_set_error(const std::string &msg) { g_err = msg; }

int gr_cuda_fail(cudaError_t e, const char *where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return GR_ECUDA;
}

extern "C" size_t gr_workspace_bytes_exact(const gr_batch *in);

extern "C" const char *gr_last_error(void) { return g_err.c_str(); }

extern "C" const char *gr_version(void) { return "grsolve 0.2 sm_100a"; }

extern "C" size_t gr_workspace_bytes(const gr_batch *in, int which) {
  if (!in || in->B < 1 || (in->W != 1 && in->W != 2)) return 0;
  if (which == 0 || which == 1) return gr_workspace_bytes_exact(in);
  if (which == 2) return 256;  // gr_mhs_greedy needs no scratch
  return 0;
}

// ---------------------------------------------------------------------------
// launch accounting + event profiling
// ---------------------------------------------------------------------------
namespace {
std::atomic<unsigned long long> g_launches{0};
std::atomic<int> g_mode{0};
std::mutex g_pmu;
struct Pending {
  std::string name;
  cudaEvent_t a, b;
};
std::vector<Pending> g_pending;
std::vector<cudaEvent_t> g_pool;
thread_local cudaEvent_t t_open = nullptr;
struct Acc {
  long long launches = 0;
  double ms = 0;
};
std::map<std::string, Acc> g_acc;

cudaEvent_t ev_get() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void drain_locked() {
  for (auto &p : g_pending) {
    float ms = 0;
    cudaEventSynchronize(p.b);
    cudaEventElapsedTime(&ms, p.a, p.b);
    Acc &a = g_acc[p.name];
    a.launches++;
    a.ms += ms;
    g_pool.push_back(p.a);
    g_pool.push_back(p.b);
  }
  g_pending.clear();
}
}  // namespace

int gr_prof_mode() { return g_mode.load(); }

void gr_prof_pre(const char *name, cudaStream_t s) {
  (void)name;
  g_launches++;
  if (!g_mode.load()) return;
  std::lock_guard<std::mutex> lk(g_pmu);
  t_open = ev_get();
  cudaEventRecord(t_open, s);
}

void gr_prof_post(const char *name, cudaStream_t s) {
  if (!g_mode.load() || !t_open) return;
  std::lock_guard<std::mutex> lk(g_pmu);
  cudaEvent_t b = ev_get();
  cudaEventRecord(b, s);
  g_pending.push_back({name, t_open, b});
  t_open = nullptr;
  if (g_pending.size() > 4096) drain_locked();
}

extern "C" unsigned long long gr_launch_count(void) { return g_launches.load(); }

extern "C" int gr_profile(int mode) {
  if (mode < 0 || mode > 2) {
    gr_set_error("gr_profile: mode must be 0, 1 or 2");
    return GR_EINVAL;
  }
  std::lock_guard<std::mutex> lk(g_pmu);
  drain_locked();
  g_acc.clear();
  unsigned long long w[8];
  gr_exact_work_read(w, 1);
  g_mode.store(mode);
  return GR_OK;
}

extern "C" int gr_profile_read(gr_kernel_stat *out, int max_stats) {
  std::lock_guard<std::mutex> lk(g_pmu);
  drain_locked();
  unsigned long long w[8] = {};
  gr_exact_work_read(w, 0);
  int n = 0;
  for (auto &kv : g_acc) {
    if (n >= max_stats) break;
    gr_kernel_stat &st = out[n++];
    memset(&st, 0, sizeof(st));
    strncpy(st.name, kv.first.c_str(), sizeof(st.name) - 1);
    st.launches = kv.second.launches;
    st.ms = kv.second.ms;
    if (kv.first == "enum_kernel" || kv.first == "queue_kernel")
      for (int i = 0; i < 8; i++) st.work[i] = w[i];
  }
  return n;
}
