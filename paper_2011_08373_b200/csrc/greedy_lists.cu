// greedy_lists.cu -- gr_mhs_greedy_lists: Johnson's greedy mhs
// over one huge phi+ given only as clause -> variable lists (CSR), without
// the variable-major bit matrix.
//
// The incremental greedy needs, per pick v*, the clauses containing v* that
// are still uncovered, and for each of them its variables (to decrement their
// counts).  The bit-matrix path reads the row R[v*] (2 MiB at C5) to find
// them, which first costs writing the whole 8 GiB matrix.  Here the
// variable -> clause lists are built on the device instead, by a counting
// sort (per-CTA histograms of the variable ids, a prefix over CTAs and
// variables, a scatter of the clause ids: ~4 bytes per literal), and each
// pick walks its own list:
//
//   counts[v] = number of clauses containing v            (the histograms)
//   repeat: v* = argmax counts (lowest index on ties; ratio rule with weights)
//           for every clause c in list(v*) not yet covered:
//               covered[c] = 1; counts[u] -= 1 for every u in c
//   until every count is 0
//
// -- the same counts and the same argmax as the textbook recount greedy, so
// the same picks (tested against the oracle on the full C5).  All picks run in
// one cooperative launch with one grid barrier per pick: the counts of pick p
// are formed on the fly as the counts of pick p-1 minus that pick's
// decrements (two count buffers, three decrement buffers, see lgreedy_kernel).  The prune (reverse-
// delete, reading R12) keeps exact per-clause hit counts over the picks'
// lists; the phi- check runs on the negative clause masks.
#include <cooperative_groups.h>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace {

constexpr int LT = 512;     // CTA size of the list kernels
constexpr int LCTA = 1184;  // histogram rows reserved in the workspace (>= the grid used)
constexpr int ST = 1024;    // CTA size of the scan

struct LCtrl {
  int done, npicks, pending, bad;
  int pad[4];
};

struct LLayout {
  size_t ctrl, hist, voff, tot, vcl, cov, counts, picks, hits, flags, smask, total;
};

LLayout llayout(const gr_clauselists *in) {
  LLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t at = o; o = align256(o + bytes); return at; };
  const size_t m = (size_t)in->m, n = (size_t)in->n_pos;
  L.ctrl = take(sizeof(LCtrl));
  L.hist = take(4 * (size_t)LCTA * m);
  L.voff = take(4 * (m + 1));
  L.tot = take(4 * m);
  L.vcl = take(4 * (size_t)std::max<int64_t>(in->nnz, 1));
  L.cov = take(std::max<size_t>(n, 1));
  L.counts = take(4 * m * 5);  // counts of two picks (ping-pong), decrements of three
  L.picks = take(4 * (m + 1));
  L.hits = take(4 * std::max<size_t>(n, 1));
  L.flags = take(4 * (m + 1));
  L.smask = take(8 * ((m + 63) / 64 + 1));
  L.total = o;
  return L;
}

struct Cand {
  u32 c, w;
  int v;
};
struct CandBetter {  // more uncovered clauses per weight; lowest index on ties (R11, R20)
  __device__ __forceinline__ Cand operator()(const Cand &a, const Cand &b) const {
    const u64 l = (u64)a.c * b.w, r = (u64)b.c * a.w;
    return (l > r || (l == r && a.v < b.v)) ? a : b;
  }
};

// ---- counting sort of the literals by variable -------------------------------
// CTA c owns the clauses [n c / G, n (c+1) / G): hist[c][v] = its literals on v
template <typename V>
__global__ void __launch_bounds__(LT) lhist_kernel(int64_t n, const int64_t *off, const V *var, int m,
                                                  u32 *hist, LCtrl *ctrl) {
  extern __shared__ u32 sh[];
  for (int v = threadIdx.x; v < m; v += LT) sh[v] = 0;
  __syncthreads();
  const int64_t j0 = n * blockIdx.x / gridDim.x, j1 = n * (blockIdx.x + 1) / gridDim.x;
  int bad = 0;
  for (int64_t e = off[j0] + threadIdx.x; e < off[j1]; e += LT) {
    const int v = (int)var[e];
    if (v < 0 || v >= m) bad = 1;
    else atomicAdd(&sh[v], 1u);
  }
  for (int64_t j = j0 + threadIdx.x; j < j1; j += LT)
    if (off[j + 1] == off[j]) bad |= 2;  // an empty clause: phi is UNSAT (R6)
  if (bad) atomicOr(&ctrl->bad, bad);
  __syncthreads();
  for (int v = threadIdx.x; v < m; v += LT) hist[(size_t)blockIdx.x * m + v] = sh[v];
}

// per variable: exclusive prefix over the CTAs (in place) and the total
__global__ void lsum_kernel(u32 *hist, int G, int m, u32 *tot, u32 *counts) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= m) return;
  u32 run = 0;
  for (int c = 0; c < G; c++) {
    const u32 t = hist[(size_t)c * m + v];
    hist[(size_t)c * m + v] = run;
    run += t;
  }
  tot[v] = run;
  counts[v] = run;  // the greedy's initial counts: clauses containing v
}

// voff = exclusive prefix of the totals over the variables (one CTA)
__global__ void __launch_bounds__(ST) lscan_kernel(const u32 *tot, int m, u32 *voff) {
  typedef cub::BlockScan<u32, ST> Scan;
  __shared__ typename Scan::TempStorage tmp;
  const int per = (m + ST - 1) / ST;
  const int i0 = min(m, (int)threadIdx.x * per), i1 = min(m, i0 + per);
  u32 s = 0;
  for (int i = i0; i < i1; i++) s += tot[i];
  u32 pre, all;
  Scan(tmp).ExclusiveSum(s, pre, all);
  for (int i = i0; i < i1; i++) {
    voff[i] = pre;
    pre += tot[i];
  }
  if (threadIdx.x == 0) voff[m] = all;
}

// scatter the clause ids into the variable lists: vcl[voff[v] + ...] = c.
// The CTA walks its clause range in tiles of LTC clauses: the tile's offsets
// and a literal -> clause map go to shared memory, then the literals are read
// coalesced and independent of each other (a thread per clause would chain
// the offset and literal loads of each clause: latency-bound).  A tile with
// more than `cap` literals falls back to a thread per clause.
constexpr int LTC = 1024;
template <typename V>
__global__ void __launch_bounds__(LT) lscatter_kernel(int64_t n, const int64_t *__restrict__ off,
                                                     const V *__restrict__ var, int m,
                                                     const u32 *__restrict__ hist, const u32 *__restrict__ voff,
                                                     u32 *__restrict__ vcl, int cap) {
  extern __shared__ u32 cur[];  // [m] the next free slot of each variable's segment of this CTA
  u32 *s_off = cur + m;         // [LTC + 1] the tile's clause offsets, relative to its first literal
  unsigned short *s_cid = (unsigned short *)(s_off + LTC + 2);  // [cap] literal -> clause of the tile
  for (int v = threadIdx.x; v < m; v += LT) cur[v] = voff[v] + hist[(size_t)blockIdx.x * m + v];
  const int64_t j0 = n * blockIdx.x / gridDim.x, j1 = n * (blockIdx.x + 1) / gridDim.x;
  for (int64_t jt = j0; jt < j1; jt += LTC) {
    const int jn = (int)min((int64_t)LTC, j1 - jt);
    const int64_t e0 = off[jt];
    __syncthreads();  // (the previous tile's map is consumed)
    for (int q = threadIdx.x; q <= jn; q += LT) s_off[q] = (u32)(off[jt + q] - e0);
    __syncthreads();
    const u32 E = s_off[jn];
    if (E > (u32)cap) {  // long clauses: a thread per clause
      for (int q = threadIdx.x; q < jn; q += LT)
        for (u32 k = s_off[q]; k < s_off[q + 1]; k++) {
          const int v = (int)var[e0 + k];
          if (v >= 0 && v < m) vcl[atomicAdd(&cur[v], 1u)] = (u32)(jt + q);
        }
      continue;
    }
    for (int q = threadIdx.x; q < jn; q += LT)
      for (u32 k = s_off[q]; k < s_off[q + 1]; k++) s_cid[k] = (unsigned short)q;
    __syncthreads();
    // 16-byte loads of the tile's literals (aligned groups of PV ids): enough
    // bytes in flight per SM to stream var at HBM rate
    constexpr int PV = 16 / (int)sizeof(V);
    const int64_t g0 = e0 / PV, g1 = (e0 + (int64_t)E + PV - 1) / PV;
    for (int64_t g = g0 + threadIdx.x; g < g1; g += LT) {
      const uint4 pk = __ldg((const uint4 *)var + g);
      const V *lit = (const V *)&pk;
#pragma unroll
      for (int i = 0; i < PV; i++) {
        const int64_t k = g * PV + i - e0;
        if (k < 0 || k >= (int64_t)E) continue;
        const int v = (int)lit[i];
        if (v >= 0 && v < m) vcl[atomicAdd(&cur[v], 1u)] = (u32)(jt + s_cid[k]);
      }
    }
  }
}

// ---- all picks in one cooperative launch ---------------------------------------
template <typename V>
__global__ void __launch_bounds__(LT) lgreedy_kernel(int m, const int64_t *__restrict__ off, const V *__restrict__ var,
                                                    const u32 *__restrict__ voff, const u32 *__restrict__ vcl,
                                                    unsigned char *cov, u32 *counts, const u32 *w,
                                                    LCtrl *ctrl, int *picks) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ u32 hist[];
  typedef cub::BlockReduce<Cand, LT> Red;
  __shared__ typename Red::TempStorage tmp;
  __shared__ int s_v;
  // counts: C[2][m] then D[3][m].  The counts of pick p are
  //   c_p(u) = C[(p-1) & 1][u] - D[(p-1) % 3][u]
  // (C[1] = the initial counts, D = 0 before pick 0); during pick p each CTA
  // stores its slice of c_p into C[p & 1] and zeroes its slice of D[(p+1) % 3],
  // and the cover of pick p adds its decrements into D[p % 3].  Every buffer a
  // pick writes was last read before the previous pick's grid barrier, and is
  // next read after this pick's: one barrier per pick.
  u32 *C = counts, *D = counts + 2 * (size_t)m;
  const int u0 = (int)((int64_t)m * blockIdx.x / gridDim.x), u1 = (int)((int64_t)m * (blockIdx.x + 1) / gridDim.x);
  int npk = 0;
  for (;;) {
    const int p = npk;
    const u32 *Cp = C + (size_t)((p + 1) & 1) * m, *Dp = D + (size_t)((p + 2) % 3) * m;
    // every CTA takes the same argmax of the same counts
    Cand best{0u, 1u, 0x7fffffff};
    for (int u = threadIdx.x; u < m; u += LT) {
      const u32 c = __ldcg(&Cp[u]) - __ldcg(&Dp[u]);
      best = CandBetter()(Cand{c, w ? w[u] : 1u, u}, best);
    }
    for (int u = u0 + threadIdx.x; u < u1; u += LT) {
      C[(size_t)(p & 1) * m + u] = __ldcg(&Cp[u]) - __ldcg(&Dp[u]);
      D[(size_t)((p + 1) % 3) * m + u] = 0u;
    }
    best = Red(tmp).Reduce(best, CandBetter());
    if (threadIdx.x == 0) {
      s_v = best.c == 0 ? -1 : best.v;
      if (blockIdx.x == 0) {
        if (best.c == 0) ctrl->done = 1;
        else picks[npk] = best.v;
        ctrl->npicks = best.c == 0 ? npk : npk + 1;
      }
    }
    for (int u = threadIdx.x; u < m; u += LT) hist[u] = 0;
    __syncthreads();
    const int v = s_v;
    if (v < 0) return;  // (every CTA saw the same counts)
    npk++;
    // cover the clauses of v's list (a slice per CTA) and count the decrements
    const u32 a = voff[v], b = voff[v + 1];
    const u32 len = b - a;
    const u32 s0 = a + (u32)((u64)len * blockIdx.x / gridDim.x);
    const u32 s1 = a + (u32)((u64)len * (blockIdx.x + 1) / gridDim.x);
    for (u32 i = s0 + threadIdx.x; i < s1; i += LT) {
      const u32 c = vcl[i];
      // the flag and the clause's bounds are loaded together (one round trip)
      const unsigned char done = __ldcg(&cov[c]);  // L2: other SMs covered it at earlier picks; each
                                                  // clause appears once in a list: no race within a pick
      const int64_t ea = off[c], eb = off[c + 1];
      if (done) continue;
      cov[c] = 1;
#pragma unroll 4
      for (int64_t e = ea; e < eb; e++) atomicAdd(&hist[(int)var[e]], 1u);
    }
    __syncthreads();
    u32 *Dq = D + (size_t)(p % 3) * m;
    for (int u = threadIdx.x; u < m; u += LT)
      if (hist[u]) atomicAdd(&Dq[u], hist[u]);
    grid.sync();
  }
}

// ---- prune (reverse-delete, R12) -------------------------------------------------
// hits[c] = number of picks whose list contains c
__global__ void lhits_kernel(const int *picks, int np, const u32 *voff, const u32 *vcl, u32 *hits) {
  for (int p = blockIdx.y; p < np; p += gridDim.y) {
    const int v = picks[p];
    const u32 a = voff[v], b = voff[v + 1];
    for (u32 i = a + blockIdx.x * blockDim.x + threadIdx.x; i < b; i += gridDim.x * blockDim.x)
      atomicAdd(&hits[vcl[i]], 1u);
  }
}
// flags[p] |= 1 if pick p (all picks when only < 0) is the sole hitter of a clause
__global__ void lprivate_kernel(const int *picks, int np, int only, const u32 *voff, const u32 *vcl,
                                const u32 *hits, int *flags) {
  const int p0 = only >= 0 ? only : 0, p1 = only >= 0 ? only + 1 : np;
  for (int p = p0 + blockIdx.y; p < p1; p += gridDim.y) {
    const int v = picks[p];
    const u32 a = voff[v], b = voff[v + 1];
    int found = 0;
    for (u32 i = a + blockIdx.x * blockDim.x + threadIdx.x; i < b && !found; i += gridDim.x * blockDim.x)
      found = __ldcg(&hits[vcl[i]]) == 1u;
    if (__syncthreads_or(found) && threadIdx.x == 0) atomicOr(&flags[p], 1);
  }
}
// drop pick x: its clauses lose one hitter
__global__ void lremove_kernel(int x, const u32 *voff, const u32 *vcl, u32 *hits) {
  const u32 a = voff[x], b = voff[x + 1];
  for (u32 i = a + blockIdx.x * blockDim.x + threadIdx.x; i < b; i += gridDim.x * blockDim.x)
    atomicSub(&hits[vcl[i]], 1u);
}
// the pruned set -> assignment words; SAT_NEG_VIOLATED if some N of phi- is inside it
__global__ void lfinal_kernel(const int *picks, int np, const int *removed, int m, const u64 *neg,
                              int n_neg, u64 *assign, int32_t *status, u64 *smask) {
  const int mw = (m + 63) / 64;
  __shared__ int s_viol;
  for (int q = threadIdx.x; q < mw; q += blockDim.x) smask[q] = 0;
  if (threadIdx.x == 0) s_viol = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < np; j += blockDim.x)
    if (!removed[j]) atomicOr((unsigned long long *)&smask[picks[j] >> 6], 1ull << (picks[j] & 63));
  __syncthreads();
  for (int q = threadIdx.x; q < mw; q += blockDim.x) assign[q] = smask[q];
  for (int j = threadIdx.x; j < n_neg; j += blockDim.x) {
    int sub = 1;
    for (int q = 0; q < mw; q++)
      if (neg[(size_t)j * mw + q] & ~smask[q]) { sub = 0; break; }
    if (sub) s_viol = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) *status = s_viol ? GR_SAT_NEG_VIOLATED : GR_SAT;
}

int validate_lists(const gr_clauselists *in) {
  if (!in) { gr_set_error("null clause lists"); return GR_EINVAL; }
  if (in->m < 1 || in->n_pos < 0 || in->nnz < 0 || in->n_neg < 0 || (in->n_neg > 0 && !in->neg) ||
      (in->n_pos > 0 && (!in->pos_off || !in->pos_var)) || (in->var_bytes != 2 && in->var_bytes != 4)) {
    gr_set_error("bad clause lists");
    return GR_EINVAL;
  }
  if ((uintptr_t)in->pos_var % 16 != 0) { gr_set_error("pos_var not 16-byte aligned"); return GR_EINVAL; }
  if (in->nnz >= (1ll << 32) || in->n_pos >= (1ll << 32)) { gr_set_error("nnz or n_pos >= 2^32"); return GR_ETOOBIG; }
  if ((size_t)in->m * 4 > 200 * 1024) { gr_set_error("m > 51200 (shared histograms)"); return GR_ETOOBIG; }
  return GR_OK;
}

PerDevice g_lattr;
int lattr() {
  return g_lattr.get([] {
    for (auto f : {(const void *)lhist_kernel<int16_t>, (const void *)lhist_kernel<int32_t>,
                   (const void *)lscatter_kernel<int16_t>, (const void *)lscatter_kernel<int32_t>,
                   (const void *)lgreedy_kernel<int16_t>, (const void *)lgreedy_kernel<int32_t>})
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024);
    return 1;
  });
}

int *pinned_lctrl() {
  static thread_local int *p = nullptr;
  if (!p && cudaMallocHost((void **)&p, sizeof(LCtrl) + 64) != cudaSuccess) p = nullptr;
  return p;
}

template <typename V>
int run_lists(const gr_clauselists *in, const LLayout &L, char *base, uint64_t *assign, int32_t *status,
              int32_t *picks_out, int32_t *n_picks, cudaStream_t st) {
  LCtrl *ctrl = (LCtrl *)(base + L.ctrl);
  u32 *hist = (u32 *)(base + L.hist), *voff = (u32 *)(base + L.voff), *tot = (u32 *)(base + L.tot);
  u32 *vcl = (u32 *)(base + L.vcl), *counts = (u32 *)(base + L.counts), *hits = (u32 *)(base + L.hits);
  unsigned char *cov = (unsigned char *)(base + L.cov);
  int *picks = (int *)(base + L.picks), *flags = (int *)(base + L.flags);
  u64 *smask = (u64 *)(base + L.smask);
  const int m = in->m;
  const int64_t n = in->n_pos;
  const V *var = (const V *)in->pos_var;
  const size_t hs = 4 * (size_t)m;
  const int sms = gr_sm_count();
  // counting-sort CTAs (GR_LSORT_PER_SM per SM; latency-bound: more in flight)
  static const int sort_per = [] {
    const char *e = getenv("GR_LSORT_PER_SM");
    const int x = e ? atoi(e) : 1;
    return (x < 1 || x > 8) ? 1 : x;
  }();
  const int G = std::min(LCTA, sort_per * sms);
  lattr();
  GR_CUDA(cudaMemsetAsync(ctrl, 0, sizeof(LCtrl), st));
  GR_CUDA(cudaMemsetAsync(cov, 0, std::max<size_t>((size_t)n, 1), st));
  GR_CUDA(cudaMemsetAsync(picks, 0xff, 4 * ((size_t)m + 1), st));
  if (n > 0) {
    GR_LAUNCH("lhist_kernel", st, lhist_kernel<V><<<G, LT, hs, st>>>(n, in->pos_off, var, m, hist, ctrl));
    GR_CUDA(cudaMemsetAsync(counts + 2 * (size_t)m, 0, 3 * hs, st));  // D = 0
    GR_LAUNCH("lsum_kernel", st, lsum_kernel<<<(m + 255) / 256, 256, 0, st>>>(hist, G, m, tot, counts + m));
    GR_LAUNCH("lscan_kernel", st, lscan_kernel<<<1, ST, 0, st>>>(tot, m, voff));
    // shared memory of the scatter: the cursors, the tile offsets, the literal map
    const size_t base_s = hs + 4 * (LTC + 2);
    const int cap = (int)std::max<int64_t>(0, std::min<int64_t>(16384, ((int64_t)220 * 1024 - (int64_t)base_s) / 2));
    GR_LAUNCH("lscatter_kernel", st,
              lscatter_kernel<V><<<G, LT, base_s + 2 * (size_t)cap, st>>>(n, in->pos_off, var, m, hist, voff, vcl, cap));
  } else {
    GR_CUDA(cudaMemsetAsync(counts, 0, 5 * hs, st));
    GR_CUDA(cudaMemsetAsync(voff, 0, 4 * ((size_t)m + 1), st));
  }
  // the picks: one cooperative launch, its grid co-resident (sized per call)
  int per = 0;
  const void *fn = (const void *)lgreedy_kernel<V>;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, LT, hs) != cudaSuccess || per < 1) {
    gr_set_error("the list greedy does not fit an SM");
    return GR_ETOOBIG;
  }
  static const int greedy_per = [] {  // CTAs per SM of the pick loop (GR_LGREEDY_PER_SM)
    const char *e = getenv("GR_LGREEDY_PER_SM");
    const int x = e ? atoi(e) : 2;
    return (x < 1 || x > 4) ? 2 : x;
  }();
  const int cgrid = sms * std::min(per, greedy_per);
  {
    const int64_t *po = in->pos_off;
    const u32 *wv = in->w;
    int mm = m;
    void *args[] = {(void *)&mm, (void *)&po, (void *)&var, (void *)&voff, (void *)&vcl, (void *)&cov,
                    (void *)&counts, (void *)&wv, (void *)&ctrl, (void *)&picks};
    gr_prof_pre("lgreedy_kernel", st);
    cudaError_t e = cudaLaunchCooperativeKernel(fn, cgrid, LT, args, hs, st);
    gr_prof_post("lgreedy_kernel", st);
    if (e != cudaSuccess) return gr_cuda_fail(e, "lgreedy_kernel");
  }
  int *h = pinned_lctrl();
  if (!h) { gr_set_error("cudaMallocHost failed"); return GR_ECUDA; }
  GR_CUDA(cudaMemcpyAsync(h, ctrl, sizeof(LCtrl), cudaMemcpyDeviceToHost, st));
  GR_CUDA(cudaStreamSynchronize(st));
  const LCtrl hc = *(const LCtrl *)h;
  const int np = hc.npicks;
  if (n_picks) *n_picks = np;
  if (hc.bad) {  // an id outside [0, m) -> bad input; an empty clause -> UNSAT (R6)
    const int32_t stv = (hc.bad & 1) ? GR_BADINPUT : GR_UNSAT;
    GR_CUDA(cudaMemsetAsync(assign, 0, 8 * (((size_t)m + 63) / 64), st));
    GR_CUDA(cudaMemcpyAsync(status, &stv, 4, cudaMemcpyHostToDevice, st));
    GR_CUDA(cudaStreamSynchronize(st));
    return GR_OK;
  }
  // prune (R12): exact hit counts over the picks' lists
  GR_CUDA(cudaMemsetAsync(hits, 0, 4 * std::max<size_t>((size_t)n, 1), st));
  GR_CUDA(cudaMemsetAsync(flags, 0, 4 * ((size_t)m + 1), st));
  std::vector<int> hpicks(np + 1), hflags(np + 1);
  if (np > 0) {
    GR_LAUNCH("lhits_kernel", st, lhits_kernel<<<dim3(16, std::min(np, 1024)), 256, 0, st>>>(picks, np, voff, vcl, hits));
    GR_LAUNCH("lprivate_kernel", st, lprivate_kernel<<<dim3(8, std::min(np, 1024)), 256, 0, st>>>(picks, np, -1, voff, vcl, hits, flags));
    GR_CUDA(cudaMemcpyAsync(hflags.data(), flags, sizeof(int) * np, cudaMemcpyDeviceToHost, st));
    GR_CUDA(cudaMemcpyAsync(hpicks.data(), picks, sizeof(int) * np, cudaMemcpyDeviceToHost, st));
    GR_CUDA(cudaStreamSynchronize(st));
  }
  // removal order: reverse pick order; with weights descending weight, equal
  // weights in reverse pick order (R12)
  std::vector<int> ord(np);
  for (int i = 0; i < np; i++) ord[i] = np - 1 - i;
  if (in->w && np > 1) {
    std::vector<uint32_t> hw(m);
    GR_CUDA(cudaMemcpyAsync(hw.data(), in->w, sizeof(uint32_t) * m, cudaMemcpyDeviceToHost, st));
    GR_CUDA(cudaStreamSynchronize(st));
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return hw[hpicks[a]] > hw[hpicks[b]]; });
  }
  std::vector<int> removed(np + 1, 0);
  int *hf = h + 8;
  for (int j : ord) {
    if (hflags[j]) continue;  // the sole hitter of some clause stays so (hit counts only decrease)
    GR_CUDA(cudaMemsetAsync(flags + j, 0, sizeof(int), st));
    GR_LAUNCH("lprivate_kernel", st, lprivate_kernel<<<dim3(64, 1), 256, 0, st>>>(picks, np, j, voff, vcl, hits, flags));
    GR_CUDA(cudaMemcpyAsync(hf, flags + j, sizeof(int), cudaMemcpyDeviceToHost, st));
    GR_CUDA(cudaStreamSynchronize(st));
    if (!*hf) {
      removed[j] = 1;
      GR_LAUNCH("lremove_kernel", st, lremove_kernel<<<64, 256, 0, st>>>(hpicks[j], voff, vcl, hits));
    }
  }
  if (np > 0) GR_CUDA(cudaMemcpyAsync(flags, removed.data(), sizeof(int) * np, cudaMemcpyHostToDevice, st));
  GR_LAUNCH("lfinal_kernel", st, lfinal_kernel<<<1, 256, 0, st>>>(picks, np, flags, m, in->neg, in->n_neg, assign,
                                                                   status, smask));
  if (picks_out) GR_CUDA(cudaMemcpyAsync(picks_out, picks, sizeof(int) * m, cudaMemcpyDeviceToDevice, st));
  GR_CUDA(cudaStreamSynchronize(st));
  return GR_OK;
}

}  // namespace

extern "C" size_t gr_greedy_lists_workspace_bytes(const gr_clauselists *in) {
  if (validate_lists(in)) return 0;
  return llayout(in).total;
}

extern "C" int gr_mhs_greedy_lists(const gr_clauselists *in, uint64_t *assign, int32_t *status,
                                   int32_t *picks, int32_t *n_picks, void *ws, size_t ws_bytes,
                                   gr_stream_t s) {
  int rc = validate_lists(in);
  if (rc) return rc;
  if (!assign || !status) { gr_set_error("null assign / status"); return GR_EINVAL; }
  const LLayout L = llayout(in);
  if (!ws || ws_bytes < L.total) { gr_set_error("workspace too small"); return GR_EWORKSPACE; }
  return in->var_bytes == 2
             ? run_lists<int16_t>(in, L, (char *)ws, assign, status, picks, n_picks, (cudaStream_t)s)
             : run_lists<int32_t>(in, L, (char *)ws, assign, status, picks, n_picks, (cudaStream_t)s);
}
