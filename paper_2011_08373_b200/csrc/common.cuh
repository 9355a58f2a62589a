// common.cuh -- shared device helpers of libgrsolve (CUDA path only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "../../include/gr.h"

typedef uint64_t u64;
typedef int64_t i64;
typedef unsigned int u32;

#define GR_KEY_NONE ((i64)0x7fffffffffffffffLL)

// ---- error plumbing (host) ------------------------------------------------
void gr_set_error(const std::string &msg);
int gr_cuda_fail(cudaError_t e, const char *where);
#define GR_CUDA(call)                                        \
  do {                                                       \
    cudaError_t _e = (call);                                 \
    if (_e != cudaSuccess) return gr_cuda_fail(_e, #call);   \
  } while (0)
#define GR_CHECK_LAUNCH(name)                                      \
  do {                                                             \
    cudaError_t _e = cudaGetLastError();                           \
    if (_e != cudaSuccess) return gr_cuda_fail(_e, name);          \
  } while (0)

// ---- launch accounting / profiling (api.cu) --------------------------------
// Every kernel launch of the library goes through GR_LAUNCH: it is counted
// (gr_launch_count) and, when profiling is on (gr_profile), bracketed by CUDA
// events recorded on the launch stream.
int gr_prof_mode();
void gr_prof_pre(const char *name, cudaStream_t s);
void gr_prof_post(const char *name, cudaStream_t s);
#define GR_LAUNCH(name, st, ...)                                   \
  do {                                                             \
    gr_prof_pre(name, st);                                         \
    __VA_ARGS__;                                                   \
    cudaError_t _e = cudaGetLastError();                           \
    gr_prof_post(name, st);                                        \
    if (_e != cudaSuccess) return gr_cuda_fail(_e, name);          \
  } while (0)
// work counters of the enumeration kernel's counting instantiation (exact.cu)
void gr_exact_work_read(unsigned long long out[8], int reset);

// ---- per-device launch settings ---------------------------------------------
// cudaFuncSetAttribute applies per device context and occupancy depends on
// the device: settings are computed once per device ordinal (thread-safe,
// std::call_once) instead of once per process.
#include <mutex>
constexpr int GR_MAX_DEVICES = 64;
inline int gr_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= GR_MAX_DEVICES) d = 0;
  return d;
}
struct PerDevice {
  std::once_flag once[GR_MAX_DEVICES];
  int val[GR_MAX_DEVICES] = {};
  // f() runs the first time the current device asks; its value is cached
  template <typename F>
  int get(F f) {
    const int d = gr_device();
    std::call_once(once[d], [&] { val[d] = f(); });
    return val[d];
  }
};
inline int gr_sm_count() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, gr_device());
  return sms > 0 ? sms : 1;
}

// ---- binomial table C(n, k), 0 <= n, k <= 64 (C(64,32) < 2^61) ------------
struct BinomTable {
  u64 v[65][65];
  constexpr BinomTable() : v() {
    for (int n = 0; n <= 64; n++) {
      v[n][0] = 1;
      for (int k = 1; k <= n; k++) v[n][k] = v[n - 1][k - 1] + (k <= n - 1 ? v[n - 1][k] : 0);
    }
  }
};
// one copy per translation unit (no relocatable device code needed)
static __device__ const BinomTable g_binom = BinomTable();

__device__ __forceinline__ u64 binom(int n, int k) {
  return (k < 0 || k > n || n < 0) ? 0ull : __ldg(&g_binom.v[n][k]);
}

// ---- generic bit helpers on 32/64-bit masks --------------------------------
__device__ __forceinline__ int popc(u32 x) { return __popc(x); }
__device__ __forceinline__ int popc(u64 x) { return __popcll(x); }
__device__ __forceinline__ int ctz(u32 x) { return __ffs(x) - 1; }
__device__ __forceinline__ int ctz(u64 x) { return __ffsll((long long)x) - 1; }
template <typename M> __device__ __forceinline__ M lowbit(M x) { return x & (~x + 1); }

// order-preserving relabel onto a support set (pext) and back (pdep), 128-bit
// support given as two words, result <= 64 bits.
__device__ __forceinline__ u64 pext128(u64 x0, u64 x1, u64 s0, u64 s1) {
  // bits of x outside the support are dropped; one step per bit of x: its
  // position among the support bits below it
  x0 &= s0;
  x1 &= s1;
  u64 r = 0;
  for (; x0; x0 &= x0 - 1) {
    const u64 l = x0 & (~x0 + 1);
    r |= 1ull << __popcll(s0 & (l - 1));
  }
  const int o = __popcll(s0);
  for (; x1; x1 &= x1 - 1) {
    const u64 l = x1 & (~x1 + 1);
    r |= 1ull << (o + __popcll(s1 & (l - 1)));
  }
  return r;
}
__device__ __forceinline__ void pdep128(u64 x, u64 s0, u64 s1, u64 &o0, u64 &o1) {
  o0 = 0;
  o1 = 0;
  int j = 0;
  while (s0) {
    u64 l = s0 & (~s0 + 1);
    if ((x >> j) & 1) o0 |= l;
    j++;
    s0 ^= l;
  }
  while (s1) {
    u64 l = s1 & (~s1 + 1);
    if ((x >> j) & 1) o1 |= l;
    j++;
    s1 ^= l;
  }
}

// colex unrank: the k-subset of {0..n-1} with rank r = sum_j C(c_j, j)
__device__ __forceinline__ u64 unrank_colex(u64 r, int k, int n) {
  u64 x = 0;
  int hi = n - 1;
  for (int j = k; j >= 1; j--) {
    // largest c in [j-1, hi] with C(c, j) <= r  (binary search)
    int lo = j - 1, h = hi;
    while (lo < h) {
      int mid = (lo + h + 1) >> 1;
      if (binom(mid, j) <= r) lo = mid; else h = mid - 1;
    }
    x |= 1ull << lo;
    r -= binom(lo, j);
    hi = lo - 1;
  }
  return x;
}

// "last block" election over a global ticket (the threadFenceReduction
// pattern): the CTA barrier orders every thread's writes before thread 0's
// gpu-scope fence (fences are cumulative), so one thread fences instead of
// every warp issuing a MEMBAR.SC.GPU.  The last CTA to arrive gets true
// (after an acquire fence) and resets the ticket.
__device__ __forceinline__ bool cta_last_arrival(unsigned *ticket, unsigned nblocks) {
  __shared__ int s_last_arrival;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const bool last = atomicAdd(ticket, 1u) == nblocks - 1;
    if (last) {
      __threadfence();
      *ticket = 0;
    }
    s_last_arrival = last;
  }
  __syncthreads();
  return s_last_arrival != 0;
}

__device__ __forceinline__ u64 sat_add(u64 a, u64 b) { u64 c = a + b; return c < a ? ~0ull : c; }

__host__ __device__ __forceinline__ size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
