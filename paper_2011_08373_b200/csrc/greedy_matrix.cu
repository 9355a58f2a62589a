// greedy_matrix.cu -- gr_mhs_greedy_matrix: Johnson's greedy mhs
// over one huge phi+ held in HBM as a variable-major bit matrix
// R[v][c/64] (bit c%64 <=> b_{v+1} in clause c), then reverse-delete to a
// minimal set (reading R12) and the phi- check.
//
// Pass t (one launch of count_kernel):   counts[v] = sum_c popc(R[v][c] & U_t[c])
//   with U_t = U_{t-1} & ~R[v*_{t-1}] computed on the fly per column tile
//   (the mark of the previous pick is fused into this pass's prologue).
// argmax_kernel:  v*_t = lowest v with the max count (R11); done when max = 0.
//
// B200 design: the pass is HBM-bound (m * n/8 bytes, ~1 op per byte).  A
// persistent CTA per SM runs a warp-specialised pipeline: one producer warp
// streams 4 KB row segments (one column tile of one row) into a 5-stage
// shared-memory ring with cp.async.bulk (TMA bulk copies, SASS UBLKCP)
// completing on mbarriers; 8 consumer warps AND each segment with the
// register-resident U tile and POPC-accumulate per-row counts in registers,
// reducing across lanes only once per work item (64 rows x 16 tiles).
#include <cooperative_groups.h>
#include <cub/block/block_reduce.cuh>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace {

constexpr int TW = 512;            // words per column tile (4 KB per row segment)
constexpr int RB = 64;             // rows per work item
constexpr int TPI = 16;            // tiles per work item
constexpr int NCW = 8;             // consumer warps
constexpr int ROWS_PER_STAGE = 8;  // one row per consumer warp
#ifndef GR_NSTAGE
#define GR_NSTAGE 5
#endif
constexpr int NSTAGE = GR_NSTAGE;
constexpr int CT = 32 * (NCW + 1); // count-kernel CTA size
constexpr size_t STAGE_BYTES = (size_t)ROWS_PER_STAGE * TW * 8;

struct GCtrl {
  int done;
  int npicks;
  int vprev;       // last pick (-1 = none): its mark is applied by the next pass
  int upar;        // U buffer parity: pass reads U[upar], writes U[upar ^ 1]
  unsigned int maxcount;
  int bad;
  // lazy greedy (lazy_step_kernel)
  int pending;     // pick whose mark the next step applies (-1 = none)
  unsigned int fresh;   // recount accumulator of the current step
  unsigned int ticket;  // last-CTA ticket of the current step
  int steps;
  int pad[2];
};

struct GLayout {
  size_t ctrl, U, counts, picks, planes, flags, smask, total;
  int nplanes;
};

int bitlen_i(long long x) {
  int b = 0;
  while (x) { b++; x >>= 1; }
  return b;
}

GLayout glayout(const gr_bitmatrix *in) {
  GLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t at = o; o = align256(o + bytes); return at; };
  const size_t ld = (size_t)in->ld;
  L.nplanes = std::max(1, bitlen_i(in->m));
  L.ctrl = take(sizeof(GCtrl));
  L.U = take(2 * ld * 8);
  L.counts = take(4 * (size_t)in->m);
  L.picks = take(4 * ((size_t)in->m + 1));
  L.planes = take((size_t)L.nplanes * ld * 8);
  L.flags = take(4 * ((size_t)in->m + 1));
  L.smask = take(8 * (((size_t)in->m + 63) / 64 + 1));
  L.total = o;
  return L;
}

// ---- PTX wrappers: mbarrier + bulk async copy ------------------------------
__device__ __forceinline__ u32 smem_u32(const void *p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64 *bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(u64 *bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(u64 *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64 *bar, u32 parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, u32 bytes, u64 *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct CountParams {
  const u64 *R;
  int64_t ld;
  int m;
  int ntiles;
  const u64 *U_in;     // U_{t-1} (or the given U for a shard count)
  u64 *U_out;          // U_t written by row-block-0 items (nullptr: no write)
  u32 *counts;
  GCtrl *ctrl;         // nullptr: no done / mark (shard count)
  int mark;            // apply U &= ~R[vprev]
};

// ---- the streaming count pass ------------------------------------------------
// Shared memory: NSTAGE row-segment stages (8 rows x 4 KB) and two tile-header
// slots (the U_{t-1} tile and the R[v*_{t-1}] tile, 4 KB each), all filled by
// the producer lane with cp.async.bulk and completed on mbarriers.
constexpr size_t TILE_BYTES = (size_t)TW * 8;
constexpr size_t HDR_BYTES = 2 * TILE_BYTES;
constexpr size_t COUNT_SMEM_V2 = NSTAGE * STAGE_BYTES + 2 * HDR_BYTES + (2 * NSTAGE + 4) * 8 + 64;

__global__ void __launch_bounds__(CT, 1) count_kernel(CountParams p) {
  extern __shared__ __align__(128) unsigned char smraw[];
  u64 *stage = (u64 *)smraw;
  u64 *hdr = (u64 *)(smraw + NSTAGE * STAGE_BYTES);   // [2][U tile | R tile]
  u64 *full = (u64 *)(smraw + NSTAGE * STAGE_BYTES + 2 * HDR_BYTES);
  u64 *empty = full + NSTAGE;
  u64 *hfull = empty + NSTAGE;   // [2]
  u64 *hempty = hfull + 2;       // [2]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int vprev = -1;
  if (p.ctrl) {
    if (*(volatile int *)&p.ctrl->done) return;
    if (p.mark) vprev = p.ctrl->vprev;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    for (int s = 0; s < 2; s++) {
      mbar_init(&hfull[s], 1);
      mbar_init(&hempty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nrb = (p.m + RB - 1) / RB;
  const int ntr = (p.ntiles + TPI - 1) / TPI;
  const int nitems = nrb * ntr;
  if (warp == NCW) {
    // ---------------- producer lane: bulk copies into the rings -----------
    if (lane == 0) {
      u32 it = 0, ht = 0;
      for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
        const int rb = item % nrb, tr = item / nrb;
        const int r0 = rb * RB;
        const int t0 = tr * TPI, t1 = min(t0 + TPI, p.ntiles);
        for (int ti = t0; ti < t1; ti++, ht++) {
          const int tw = (int)min((int64_t)TW, p.ld - (int64_t)ti * TW);
          // tile header: U_{t-1} tile (+ R[v*] tile when marking)
          const int hs = ht & 1;
          mbar_wait(&hempty[hs], ((ht >> 1) & 1) ^ 1);
          u64 *h = hdr + (size_t)hs * (HDR_BYTES / 8);
          mbar_expect_tx(&hfull[hs], (u32)((vprev >= 0 ? 2 : 1) * tw * 8));
          bulk_g2s(h, p.U_in + (size_t)ti * TW, (u32)(tw * 8), &hfull[hs]);
          if (vprev >= 0)
            bulk_g2s(h + TW, p.R + (size_t)vprev * p.ld + (size_t)ti * TW, (u32)(tw * 8), &hfull[hs]);
          for (int g = 0; g < RB / ROWS_PER_STAGE; g++, it++) {
            const int s = it % NSTAGE;
            mbar_wait(&empty[s], ((it / NSTAGE) & 1) ^ 1);
            int nrow = min(ROWS_PER_STAGE, p.m - (r0 + g * ROWS_PER_STAGE));
            nrow = max(nrow, 0);
            mbar_expect_tx(&full[s], (u32)(nrow * tw * 8));
            for (int w = 0; w < nrow; w++) {
              const int row = r0 + g * ROWS_PER_STAGE + w;
              bulk_g2s(stage + (size_t)s * ROWS_PER_STAGE * TW + (size_t)w * TW,
                       p.R + (size_t)row * p.ld + (size_t)ti * TW, (u32)(tw * 8), &full[s]);
            }
          }
        }
      }
    }
    return;
  }
  // ---------------- consumer warps ------------------------------------------
  u32 it = 0, ht = 0;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int rb = item % nrb, tr = item / nrb;
    const int r0 = rb * RB;
    const int t0 = tr * TPI, t1 = min(t0 + TPI, p.ntiles);
    u32 acc[RB / ROWS_PER_STAGE];
#pragma unroll
    for (int g = 0; g < RB / ROWS_PER_STAGE; g++) acc[g] = 0;
    for (int ti = t0; ti < t1; ti++, ht++) {
      const int tw = (int)min((int64_t)TW, p.ld - (int64_t)ti * TW);
      const int nstep = tw / 64;
      // U_t fragment of this lane (words s*64 + 2*lane + {0,1} of the tile)
      const int hs = ht & 1;
      mbar_wait(&hfull[hs], (ht >> 1) & 1);
      const u64 *h = hdr + (size_t)hs * (HDR_BYTES / 8);
      ulonglong2 u[TW / 64];
#pragma unroll
      for (int s = 0; s < TW / 64; s++) {
        if (s < nstep) {
          ulonglong2 x = *(const ulonglong2 *)(h + s * 64 + 2 * lane);
          if (vprev >= 0) {
            const ulonglong2 r = *(const ulonglong2 *)(h + TW + s * 64 + 2 * lane);
            x.x &= ~r.x;
            x.y &= ~r.y;
          }
          u[s] = x;
          if (p.U_out && rb == 0 && warp == 0)
            *(ulonglong2 *)(p.U_out + (size_t)ti * TW + (size_t)s * 64 + 2 * lane) = x;
        } else {
          u[s] = make_ulonglong2(0, 0);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&hempty[hs]);
#pragma unroll
      for (int g = 0; g < RB / ROWS_PER_STAGE; g++, it++) {
        const int s = it % NSTAGE;
        mbar_wait(&full[s], (it / NSTAGE) & 1);
        const int row = r0 + g * ROWS_PER_STAGE + warp;
        if (row < p.m) {
          const u64 *seg = stage + (size_t)s * ROWS_PER_STAGE * TW + (size_t)warp * TW;
          u32 c = 0;
#pragma unroll
          for (int q = 0; q < TW / 64; q++) {
            if (q < nstep) {
              const ulonglong2 d = *(const ulonglong2 *)(seg + q * 64 + 2 * lane);
              c += __popcll(d.x & u[q].x) + __popcll(d.y & u[q].y);
            }
          }
          acc[g] += c;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
    }
    // one reduction per row per item
#pragma unroll
    for (int g = 0; g < RB / ROWS_PER_STAGE; g++) {
      u32 v = acc[g];
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      const int row = r0 + g * ROWS_PER_STAGE + warp;
      if (lane == 0 && row < p.m && v) atomicAdd(&p.counts[row], v);
    }
  }
}

// ---- argmax + bookkeeping (one CTA) ------------------------------------------
// The pick maximises count[v] / w[v] (w = 1 without weights: the plain
// argmax), compared exactly as c_a * w_b > c_b * w_a, lowest index on ties
// (readings R11, R20).
struct Cand {
  u32 c, w;
  int v;
};
struct CandBetter {
  __device__ __forceinline__ Cand operator()(const Cand &a, const Cand &b) const {
    const u64 l = (u64)a.c * b.w, r = (u64)b.c * a.w;
    return (l > r || (l == r && a.v < b.v)) ? a : b;
  }
};
constexpr int AT = 1024;
__global__ void __launch_bounds__(AT) argmax_kernel(u32 *counts, int m, const u32 *w, GCtrl *ctrl,
                                                    int *picks) {
  typedef cub::BlockReduce<Cand, AT> Red;
  __shared__ typename Red::TempStorage tmp;
  if (*(volatile int *)&ctrl->done) return;
  Cand best{0u, 1u, 0x7fffffff};
  for (int v = threadIdx.x; v < m; v += AT) {
    const Cand cv{counts[v], w ? w[v] : 1u, v};
    counts[v] = 0;  // ready for the next pass
    best = CandBetter()(cv, best);
  }
  best = Red(tmp).Reduce(best, CandBetter());
  if (threadIdx.x == 0) {
    ctrl->maxcount = best.c;
    ctrl->upar ^= 1;  // the pass just run wrote U[upar ^ 1]
    if (best.c == 0) {
      ctrl->done = 1;
      ctrl->vprev = -1;
    } else {
      picks[ctrl->npicks] = best.v;
      ctrl->npicks += 1;
      ctrl->vprev = best.v;
    }
  }
}

__global__ void init_kernel(u64 *U0, int64_t ld, int64_t n, GCtrl *ctrl, u32 *counts, int m,
                            int *picks) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t w = i; w < ld; w += stride) {
    const int64_t c0 = w * 64;
    u64 x = 0;
    if (c0 + 64 <= n) x = ~0ull;
    else if (c0 < n) x = (1ull << (n - c0)) - 1;
    U0[w] = x;
  }
  for (int64_t v = i; v < m; v += stride) { counts[v] = 0; picks[v] = -1; }
  if (i == 0) {
    ctrl->done = 0;
    ctrl->npicks = 0;
    ctrl->vprev = -1;
    ctrl->upar = 0;
    ctrl->maxcount = 0;
    ctrl->bad = 0;
    ctrl->pending = -1;
    ctrl->fresh = 0;
    ctrl->ticket = 0;
    ctrl->steps = 0;
  }
}

// ---- incremental greedy -----------------------------------
// With the clause-major variable lists (CSR) at hand the counts are kept exact
// without re-streaming the matrix: count[v] starts as the number of clauses
// containing v (a histogram of the CSR), and when v* is picked every newly
// covered clause c (U ∩ R[v*], one 2 MiB row) decrements the count of each of
// its variables.  Picks are identical to the recounting loop (same counts,
// same lowest-index argmax); the bytes per pick drop from m·n/8 to about
// n/8 + |newly covered|·(clause length + 1)·(var bytes).
template <typename V>
__global__ void csr_hist_kernel(int64_t n, const int64_t *off, const V *var, int m, u32 *counts) {
  extern __shared__ u32 hist[];
  for (int v = threadIdx.x; v < m; v += blockDim.x) hist[v] = 0;
  __syncthreads();
  const int64_t e0 = off[0], e1 = off[n];
  for (int64_t e = e0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < e1;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&hist[(int)var[e]], 1u);
  __syncthreads();
  for (int v = threadIdx.x; v < m; v += blockDim.x)
    if (hist[v]) atomicAdd(&counts[v], hist[v]);
}

constexpr int IT = 512;
// the argmax of the counts (lowest index on ties) -> ctrl (pick or done)
__device__ __forceinline__ void pick_argmax(const u32 *counts, int m, const u32 *w, GCtrl *ctrl,
                                            int *picks) {
  typedef cub::BlockReduce<Cand, IT> Red;
  __shared__ typename Red::TempStorage tmp;
  Cand best{0u, 1u, 0x7fffffff};
  for (int v = threadIdx.x; v < m; v += IT)
    best = CandBetter()(Cand{__ldcg(&counts[v]), w ? w[v] : 1u, v}, best);
  best = Red(tmp).Reduce(best, CandBetter());
  if (threadIdx.x == 0) {
    if (best.c == 0) {  // every count is 0: U is empty
      ctrl->done = 1;
      ctrl->pending = -1;
    } else {
      picks[ctrl->npicks] = best.v;
      ctrl->npicks += 1;
      ctrl->pending = best.v;
    }
  }
}

__global__ void __launch_bounds__(IT) first_pick_kernel(const u32 *counts, int m, const u32 *w,
                                                       GCtrl *ctrl, int *picks) {
  pick_argmax(counts, m, w, ctrl, picks);
}

// one pick: apply the pending pick v (cover its clauses, decrement counts),
// then the last CTA chooses the next pick
template <typename V, bool PICK = true>
__global__ void __launch_bounds__(IT) incr_step_kernel(const u64 *R, int64_t ld, int m, u64 *U,
                                                      u32 *counts, const int64_t *off,
                                                      const V *var, const u32 *w, GCtrl *ctrl,
                                                      int *picks) {
  extern __shared__ u32 hist[];
  if (*(volatile int *)&ctrl->done) return;
  const int v = ctrl->pending;
  for (int u = threadIdx.x; u < m; u += IT) hist[u] = 0;
  __syncthreads();
  const int64_t a = ld * blockIdx.x / gridDim.x, b = ld * (blockIdx.x + 1) / gridDim.x;
  const u64 *Rv = R + (size_t)v * ld;
  for (int64_t w = a + threadIdx.x; w < b; w += IT) {
    const u64 r = Rv[w];
    if (!r) continue;
    const u64 u = U[w];
    u64 nw = u & r;  // clauses newly covered by v
    if (!nw) continue;
    U[w] = u & ~r;
    while (nw) {
      const int64_t c = w * 64 + (__ffsll((long long)nw) - 1);
      nw &= nw - 1;
      for (int64_t e = off[c]; e < off[c + 1]; e++) atomicAdd(&hist[(int)var[e]], 1u);
    }
  }
  __syncthreads();
  for (int u = threadIdx.x; u < m; u += IT)
    if (hist[u]) atomicSub(&counts[u], hist[u]);
  if (!PICK) return;  // sharded greedy: the next pick needs the all-reduced counts
  if (cta_last_arrival(&ctrl->ticket, gridDim.x)) {
    pick_argmax(counts, m, w, ctrl, picks);
    if (threadIdx.x == 0) ctrl->steps += 1;
  }
}

// ---- column-sharded greedy ----------------------------------
// Each rank owns a range of clause columns; the host all-reduces (SUM) the
// per-rank counts between steps, so every rank takes the same pick from the
// same global counts.  One step: pick from the global counts, then cover this
// shard's clauses of the pick and bring the local counts up to date
// (incremental decrement, or mark + recount pass).
__global__ void __launch_bounds__(IT) shard_pick_kernel(const u32 *gcounts, int m, const u32 *w,
                                                       GCtrl *ctrl, int *picks, u32 *counts,
                                                       int zero_counts) {
  typedef cub::BlockReduce<Cand, IT> Red;
  __shared__ typename Red::TempStorage tmp;
  if (*(volatile int *)&ctrl->done) return;
  Cand best{0u, 1u, 0x7fffffff};
  for (int v = threadIdx.x; v < m; v += IT) {
    best = CandBetter()(Cand{gcounts[v], w ? w[v] : 1u, v}, best);
    if (zero_counts) counts[v] = 0;  // the recount pass accumulates into them
  }
  best = Red(tmp).Reduce(best, CandBetter());
  if (threadIdx.x == 0) {
    ctrl->maxcount = best.c;
    if (best.c == 0) {  // no uncovered clause anywhere
      ctrl->done = 1;
      ctrl->pending = ctrl->vprev = -1;
    } else {
      picks[ctrl->npicks] = best.v;
      ctrl->npicks += 1;
      ctrl->pending = ctrl->vprev = best.v;
    }
  }
}

// U &= ~R[v*] on this shard (recounting steps)
__global__ void shard_mark_kernel(const u64 *R, int64_t ld, u64 *U, const GCtrl *ctrl) {
  if (*(volatile const int *)&ctrl->done) return;
  const int v = ctrl->vprev;
  const u64 *Rv = R + (size_t)v * ld;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < ld;
       w += (int64_t)gridDim.x * blockDim.x)
    U[w] &= ~Rv[w];
}

// the whole incremental greedy in one cooperative launch: per pick, every CTA
// covers its slice of R[v] and decrements (shared histogram), a grid barrier,
// then every CTA takes the same argmax of the counts (identical reads), a
// second barrier before the counts change again.  CTA 0 records the pick.
template <typename V>
__global__ void __launch_bounds__(IT) incr_all_kernel(const u64 *R, int64_t ld, int m, u64 *U,
                                                     u32 *counts, const int64_t *off,
                                                     const V *var, const u32 *w, GCtrl *ctrl,
                                                     int *picks) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ u32 hist[];
  typedef cub::BlockReduce<Cand, IT> Red;
  __shared__ typename Red::TempStorage tmp;
  __shared__ int s_v;
  if (threadIdx.x == 0) s_v = ctrl->done ? -1 : ctrl->pending;
  __syncthreads();
  int npk = ctrl->npicks;
  const int64_t a = ld * blockIdx.x / gridDim.x, b = ld * (blockIdx.x + 1) / gridDim.x;
  while (s_v >= 0) {
    const int v = s_v;
    for (int u = threadIdx.x; u < m; u += IT) hist[u] = 0;
    __syncthreads();
    const u64 *Rv = R + (size_t)v * ld;
    for (int64_t wd = a + threadIdx.x; wd < b; wd += IT) {
      const u64 r = Rv[wd];
      if (!r) continue;
      const u64 uu = U[wd];
      u64 nw = uu & r;  // clauses newly covered by v
      if (!nw) continue;
      U[wd] = uu & ~r;
      while (nw) {
        const int64_t c = wd * 64 + (__ffsll((long long)nw) - 1);
        nw &= nw - 1;
        for (int64_t e = off[c]; e < off[c + 1]; e++) atomicAdd(&hist[(int)var[e]], 1u);
      }
    }
    __syncthreads();
    for (int u = threadIdx.x; u < m; u += IT)
      if (hist[u]) atomicSub(&counts[u], hist[u]);
    grid.sync();
    Cand best{0u, 1u, 0x7fffffff};
    for (int u = threadIdx.x; u < m; u += IT)
      best = CandBetter()(Cand{__ldcg(&counts[u]), w ? w[u] : 1u, u}, best);
    best = Red(tmp).Reduce(best, CandBetter());
    if (threadIdx.x == 0) {
      s_v = best.c == 0 ? -1 : best.v;
      if (blockIdx.x == 0) {
        if (best.c == 0) {
          ctrl->done = 1;
          ctrl->pending = -1;
        } else {
          picks[npk] = best.v;
          ctrl->pending = best.v;
        }
        ctrl->npicks = best.c == 0 ? npk : npk + 1;
      }
    }
    if (best.c != 0) npk++;
    grid.sync();  // every CTA has read the counts
  }
}

// ---- prune: bit-sliced hit counters over the picks ----------------------------
// planes[i][w] is bit i of the per-clause hit count; add/sub ripple carries.
__global__ void planes_build_kernel(const u64 *R, int64_t ld, const int *picks, const GCtrl *ctrl,
                                    u64 *planes, int nplanes) {
  const int np = ctrl->npicks;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < ld;
       w += (int64_t)gridDim.x * blockDim.x) {
    u64 P[32];
    for (int i = 0; i < nplanes; i++) P[i] = 0;
    for (int j = 0; j < np; j++) {
      u64 carry = R[(size_t)picks[j] * ld + w];
      for (int i = 0; i < nplanes && carry; i++) {
        const u64 t = P[i] & carry;
        P[i] ^= carry;
        carry = t;
      }
    }
    for (int i = 0; i < nplanes; i++) planes[(size_t)i * ld + w] = P[i];
  }
}

// one[w] = clauses hit exactly once (bit 0 set, all higher planes clear)
__global__ void one_kernel(const u64 *planes, int nplanes, int64_t ld, u64 *one) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < ld;
       w += (int64_t)gridDim.x * blockDim.x) {
    u64 hi = 0;
    for (int i = 1; i < nplanes; i++) hi |= planes[(size_t)i * ld + w];
    one[w] = planes[w] & ~hi;
  }
}

// flags[j] |= 1 if pick j (all picks when only < 0, else pick `only`) is the
// sole hitter of some clause
__global__ void private_kernel(const u64 *R, int64_t ld, const int *picks, const GCtrl *ctrl,
                               const u64 *one, int *flags, int only) {
  const int np = ctrl->npicks;
  const int j0 = only >= 0 ? only : 0, j1 = only >= 0 ? only + 1 : np;
  for (int j = j0; j < j1; j++) {
    const u64 *row = R + (size_t)picks[j] * ld;
    int found = 0;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < ld;
         w += (int64_t)gridDim.x * blockDim.x)
      if (row[w] & one[w]) { found = 1; break; }
    if (__syncthreads_or(found) && threadIdx.x == 0) atomicOr(&flags[j], 1);
  }
}

// drop pick x: subtract its row from the bit-sliced counters, refresh one[]
__global__ void remove_kernel(const u64 *R, int64_t ld, int x, u64 *planes, int nplanes, u64 *one) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < ld;
       w += (int64_t)gridDim.x * blockDim.x) {
    u64 borrow = R[(size_t)x * ld + w];
    if (!borrow) continue;
    for (int i = 0; i < nplanes && borrow; i++) {
      const u64 p = planes[(size_t)i * ld + w];
      const u64 t = ~p & borrow;
      planes[(size_t)i * ld + w] = p ^ borrow;
      borrow = t;
    }
    u64 hi = 0;
    for (int i = 1; i < nplanes; i++) hi |= planes[(size_t)i * ld + w];
    one[w] = planes[w] & ~hi;
  }
}

__global__ void finalize_kernel(const int *picks, const GCtrl *ctrl, const int *removed, int m,
                                const u64 *neg, int n_neg, u64 *assign, int32_t *status,
                                u64 *smask) {
  const int mw = (m + 63) / 64;
  const int np = ctrl->npicks;
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

// ---- CSR packing ------------------------------------------------------------------
template <typename V>
__global__ void pack_vm_kernel(int m, int64_t n, const int64_t *off, const V *var, u64 *bits,
                               int64_t ld, int32_t *bad, int varmajor) {
  const int mw = (m + 63) / 64;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = off[c], e1 = off[c + 1];
    if (e1 <= e0 && bad) atomicOr(bad, 2);
    for (int64_t e = e0; e < e1; e++) {
      const int v = (int)var[e];
      if (v < 0 || v >= m) {
        if (bad) atomicOr(bad, 1);
        continue;
      }
      unsigned long long old, bit;
      if (varmajor) {
        bit = 1ull << (c & 63);
        old = atomicOr((unsigned long long *)&bits[(size_t)v * ld + (c >> 6)], bit);
      } else {
        bit = 1ull << (v & 63);
        old = atomicOr((unsigned long long *)&bits[(size_t)c * mw + (v >> 6)], bit);
      }
      if ((old & bit) && bad) atomicOr(bad, 4);  // the clause lists v twice
    }
  }
}

// Tiled var-major pack: a CTA owns a tile of PK_R rows x PK_C clauses (16
// words = one 128-byte line per row), builds it in shared memory with shared
// atomics (flagging out-of-range / empty / repeated ids) and writes every
// row's line once -- every word of the matrix is written (zeros included), so
// the caller need not clear it.  Each clause list is read once per row block.
constexpr int PK_T = 512;
constexpr int PK_R = 1024;            // rows per tile
constexpr int PK_W = 16;              // words per tile row (1024 clauses)
constexpr size_t PK_SMEM = (size_t)PK_R * PK_W * 8;  // 128 KB
template <typename V>
__global__ void __launch_bounds__(PK_T) pack_vm_tiled_kernel(int m, int64_t n, const int64_t *off,
                                                            const V *var, u64 *bits, int64_t ld,
                                                            int32_t *bad) {
  extern __shared__ unsigned long long tile[];  // [PK_R][PK_W]
  const int nrb = (m + PK_R - 1) / PK_R;
  const int64_t ncb = ld / PK_W;
  int flags = 0;
  for (int64_t g = blockIdx.x; g < (int64_t)nrb * ncb; g += gridDim.x) {
    const int rb = (int)(g % nrb);
    const int64_t cb = g / nrb;
    const int r0 = rb * PK_R;
    const int nr = min(PK_R, m - r0);
    for (int q = threadIdx.x; q < PK_R * PK_W; q += PK_T) tile[q] = 0;
    __syncthreads();
    for (int cc = threadIdx.x; cc < PK_W * 64; cc += PK_T) {
      const int64_t c = cb * (PK_W * 64) + cc;
      if (c >= n) break;
      const int64_t e0 = off[c], e1 = off[c + 1];
      if (rb == 0 && e1 <= e0) flags |= 2;
      const unsigned long long bit = 1ull << (cc & 63);
      for (int64_t e = e0; e < e1; e++) {
        const int v = (int)var[e];
        if (v < 0 || v >= m) {
          if (rb == 0) flags |= 1;
          continue;
        }
        if (v < r0 || v >= r0 + nr) continue;
        if (atomicOr(&tile[(v - r0) * PK_W + (cc >> 6)], bit) & bit) flags |= 4;
      }
    }
    __syncthreads();
    // write: 8 threads per row, 16 bytes each -> one 128-byte line per row
    for (int q = threadIdx.x; q < nr * (PK_W / 2); q += PK_T) {
      const int r = q / (PK_W / 2), h = q % (PK_W / 2);
      ulonglong2 *dst = (ulonglong2 *)(bits + (size_t)(r0 + r) * ld + cb * PK_W) + h;
      *dst = make_ulonglong2(tile[r * PK_W + 2 * h], tile[r * PK_W + 2 * h + 1]);
    }
    __syncthreads();
  }
  if (bad && flags) atomicOr(bad, flags);
}

// the count pass grid (one persistent CTA per SM); sets the kernels' dynamic
// shared memory limits on first use of each device
PerDevice g_count_grid;
int count_grid() {
  return g_count_grid.get([] {
    cudaFuncSetAttribute(count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)COUNT_SMEM_V2);
    for (auto f : {(const void *)incr_step_kernel<int16_t>, (const void *)incr_step_kernel<int32_t>,
                   (const void *)csr_hist_kernel<int16_t>, (const void *)csr_hist_kernel<int32_t>,
                   (const void *)incr_all_kernel<int16_t>, (const void *)incr_all_kernel<int32_t>})
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (auto f : {(const void *)pack_vm_tiled_kernel<int16_t>, (const void *)pack_vm_tiled_kernel<int32_t>})
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PK_SMEM);
    return gr_sm_count();
  });
}

int validate_matrix(const gr_bitmatrix *in) {
  if (!in || !in->bits) { gr_set_error("null matrix"); return GR_EINVAL; }
  if (in->m < 1 || in->n_pos < 0 || in->n_neg < 0 || (in->n_neg > 0 && !in->neg)) {
    gr_set_error("bad matrix sizes");
    return GR_EINVAL;
  }
  if (in->pos_off && in->pos_var && in->var_bytes != 2 && in->var_bytes != 4) {
    gr_set_error("var_bytes must be 2 or 4");
    return GR_EINVAL;
  }
  if (in->ld < (in->n_pos + 63) / 64 || in->ld % 64 != 0 || in->ld < 64) {
    gr_set_error("ld must be >= ceil(n_pos/64), >= 64 and a multiple of 64");
    return GR_EINVAL;
  }
  return GR_OK;
}

int *pinned_ctrl() {
  static thread_local int *p = nullptr;
  if (!p && cudaMallocHost((void **)&p, sizeof(GCtrl) + 64) != cudaSuccess) p = nullptr;
  return p;
}

}  // namespace

extern "C" int64_t gr_bitmatrix_ld(int64_t n_pos) {
  int64_t w = (n_pos + 63) / 64;
  w = (w + 63) / 64 * 64;
  return w < 64 ? 64 : w;
}

extern "C" int gr_pack_varmajor(int32_t m, int64_t n, const int64_t *off, const void *var,
                                int var_bytes, uint64_t *bits, int64_t ld, int32_t *d_bad,
                                gr_stream_t s) {
  if (m < 1 || n < 0 || !off || (!var && n > 0) || !bits || ld < (n + 63) / 64 ||
      (var_bytes != 2 && var_bytes != 4)) {
    gr_set_error("gr_pack_varmajor: bad arguments");
    return GR_EINVAL;
  }
  if (n == 0) return GR_OK;
  cudaStream_t st = (cudaStream_t)s;
  if (ld % PK_W == 0) {
    const int grid = count_grid();  // one CTA per SM (also sets the smem attribute)
    if (var_bytes == 2)
      GR_LAUNCH("pack_vm_tiled_kernel", st, pack_vm_tiled_kernel<int16_t><<<grid, PK_T, PK_SMEM, st>>>(m, n, off, (const int16_t *)var, bits, ld, d_bad));
    else
      GR_LAUNCH("pack_vm_tiled_kernel", st, pack_vm_tiled_kernel<int32_t><<<grid, PK_T, PK_SMEM, st>>>(m, n, off, (const int32_t *)var, bits, ld, d_bad));
    return GR_OK;
  }
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  if (var_bytes == 2)
    GR_LAUNCH("pack_vm_kernel", (cudaStream_t)s, pack_vm_kernel<int16_t><<<grid, 256, 0, (cudaStream_t)s>>>(m, n, off, (const int16_t *)var, bits, ld, d_bad, 1));
  else
    GR_LAUNCH("pack_vm_kernel", (cudaStream_t)s, pack_vm_kernel<int32_t><<<grid, 256, 0, (cudaStream_t)s>>>(m, n, off, (const int32_t *)var, bits, ld, d_bad, 1));
  return GR_OK;
}

extern "C" int gr_pack_clausemajor(int32_t m, int64_t n, const int64_t *off, const void *var,
                                   int var_bytes, uint64_t *masks, int32_t *d_bad, gr_stream_t s) {
  if (m < 1 || n < 0 || !off || (!var && n > 0) || !masks || (var_bytes != 2 && var_bytes != 4)) {
    gr_set_error("gr_pack_clausemajor: bad arguments");
    return GR_EINVAL;
  }
  if (n == 0) return GR_OK;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  if (var_bytes == 2)
    GR_LAUNCH("pack_cm_kernel", (cudaStream_t)s, pack_vm_kernel<int16_t><<<grid, 256, 0, (cudaStream_t)s>>>(m, n, off, (const int16_t *)var, masks, 0, d_bad, 0));
  else
    GR_LAUNCH("pack_cm_kernel", (cudaStream_t)s, pack_vm_kernel<int32_t><<<grid, 256, 0, (cudaStream_t)s>>>(m, n, off, (const int32_t *)var, masks, 0, d_bad, 0));
  return GR_OK;
}

extern "C" size_t gr_greedy_matrix_workspace_bytes(const gr_bitmatrix *in) {
  if (validate_matrix(in)) return 0;
  return glayout(in).total;
}

extern "C" int gr_greedy_count_shard(const gr_bitmatrix *shard, const uint64_t *d_U,
                                     uint32_t *d_counts, gr_stream_t s) {
  int rc = validate_matrix(shard);
  if (rc) return rc;
  if (!d_U || !d_counts) { gr_set_error("null U / counts"); return GR_EINVAL; }
  cudaStream_t st = (cudaStream_t)s;
  GR_CUDA(cudaMemsetAsync(d_counts, 0, sizeof(u32) * shard->m, st));
  CountParams p{shard->bits, shard->ld, shard->m, (int)((shard->ld + TW - 1) / TW), d_U, nullptr,
                d_counts, nullptr, 0};
  GR_LAUNCH("count_kernel", (cudaStream_t)s, count_kernel<<<count_grid(), CT, COUNT_SMEM_V2, st>>>(p));
  return GR_OK;
}

// prune order of the picks (positions into picks[0..np)): reverse pick
// order; with weights descending weight, equal weights in reverse pick order
// (reading R12)
static int removal_order(const gr_bitmatrix *in, const std::vector<int> &hpicks, int np, cudaStream_t st,
                  std::vector<int> &ord) {
  ord.resize(np);
  for (int i = 0; i < np; i++) ord[i] = np - 1 - i;
  if (!in->w || np < 2) return GR_OK;
  std::vector<uint32_t> hw(in->m);
  GR_CUDA(cudaMemcpyAsync(hw.data(), in->w, sizeof(uint32_t) * in->m, cudaMemcpyDeviceToHost, st));
  GR_CUDA(cudaStreamSynchronize(st));
  std::stable_sort(ord.begin(), ord.end(),
                   [&](int a, int b) { return hw[hpicks[a]] > hw[hpicks[b]]; });
  return GR_OK;
}

extern "C" int gr_mhs_greedy_matrix(const gr_bitmatrix *in, uint64_t *assign, int32_t *status,
                                    int32_t *picks, int32_t *n_picks, void *ws, size_t ws_bytes,
                                    gr_stream_t s) {
  int rc = validate_matrix(in);
  if (rc) return rc;
  if (!assign || !status) { gr_set_error("null assign / status"); return GR_EINVAL; }
  GLayout L = glayout(in);
  if (!ws || ws_bytes < L.total) { gr_set_error("workspace too small"); return GR_EWORKSPACE; }
  char *base = (char *)ws;
  GCtrl *ctrl = (GCtrl *)(base + L.ctrl);
  u64 *U = (u64 *)(base + L.U);
  u32 *counts = (u32 *)(base + L.counts);
  int *wpicks = (int *)(base + L.picks);
  u64 *planes = (u64 *)(base + L.planes);
  int *flags = (int *)(base + L.flags);
  u64 *smask = (u64 *)(base + L.smask);
  cudaStream_t st = (cudaStream_t)s;
  const int64_t ld = in->ld;
  const int ntiles = (int)((ld + TW - 1) / TW);
  GR_LAUNCH("init_kernel", (cudaStream_t)s, init_kernel<<<592, 256, 0, st>>>(U, ld, in->n_pos, ctrl, counts, in->m, wpicks));
  const int grid = count_grid();
  int *h = pinned_ctrl();
  if (!h) { gr_set_error("cudaMallocHost failed"); return GR_ECUDA; }
  const int CHUNK = 8;
  int t = 0;
  bool eager = in->pos_off == nullptr || in->pos_var == nullptr || in->m > 50000 ||
               getenv("GR_GREEDY_EAGER") != nullptr;
  if (!eager) {
    // incremental greedy: CSR histogram, then one cover-and-decrement step per pick
    const int hgrid = (int)std::min<int64_t>((in->n_pos * 9 + 255) / 256, 148 * 8);
    const size_t hs = sizeof(u32) * (size_t)in->m;
    if (in->var_bytes == 2)
      GR_LAUNCH("csr_hist_kernel", st, csr_hist_kernel<int16_t><<<std::max(hgrid, 1), 256, hs, st>>>(
                                          in->n_pos, in->pos_off, (const int16_t *)in->pos_var, in->m, counts));
    else
      GR_LAUNCH("csr_hist_kernel", st, csr_hist_kernel<int32_t><<<std::max(hgrid, 1), 256, hs, st>>>(
                                          in->n_pos, in->pos_off, (const int32_t *)in->pos_var, in->m, counts));
    GR_LAUNCH("first_pick_kernel", st, first_pick_kernel<<<1, IT, 0, st>>>(counts, in->m, in->w, ctrl, wpicks));
    bool coop_done = false;
    {
      // one cooperative launch for all picks: its grid must be co-resident, so
      // it is sized per call from the occupancy at this call's shared memory
      // (hs = 4 m bytes) on this device -- 0 falls back to per-pick launches
      count_grid();  // sets the dynamic shared memory limits on this device
      int per = 0, coop = 0;
      cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, gr_device());
      const void *fn = in->var_bytes == 2 ? (const void *)incr_all_kernel<int16_t>
                                          : (const void *)incr_all_kernel<int32_t>;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, IT, hs) != cudaSuccess) per = 0;
      static const bool no_coop = getenv("GR_NO_COOP") != nullptr;
      const int cgrid = (coop && per > 0 && !no_coop) ? gr_sm_count() * std::min(per, 2) : 0;
      if (cgrid > 0) {
        const int64_t ldv = ld;
        const int mv = in->m;
        void *args[] = {(void *)&in->bits, (void *)&ldv, (void *)&mv, (void *)&U, (void *)&counts,
                        (void *)&in->pos_off, (void *)&in->pos_var, (void *)&in->w, (void *)&ctrl,
                        (void *)&wpicks};
        gr_prof_pre("incr_all_kernel", st);
        cudaError_t e = cudaLaunchCooperativeKernel(fn, cgrid, IT, args, hs, st);
        gr_prof_post("incr_all_kernel", st);
        if (e == cudaErrorCooperativeLaunchTooLarge) {
          cudaGetLastError();  // not co-resident after all: per-pick launches below
        } else {
          if (e != cudaSuccess) return gr_cuda_fail(e, "incr_all_kernel");
          GR_CUDA(cudaMemcpyAsync(h, ctrl, sizeof(GCtrl), cudaMemcpyDeviceToHost, st));
          GR_CUDA(cudaStreamSynchronize(st));
          coop_done = ((GCtrl *)h)->done != 0;
        }
      }
    }
    const int STEPS = 32;
    static const int igrid_env = [] {  // CTAs of the incremental step (GR_INCR_GRID)
      const char *e = getenv("GR_INCR_GRID");
      return e ? atoi(e) : 0;
    }();
    int igrid = igrid_env ? igrid_env : 2 * grid;  // two per SM: measured 10.8 -> 7.7 ms on C5
    if (igrid < 1 || igrid > 4 * grid) igrid = grid;
    for (int round = 0; !coop_done; round++) {
      for (int j = 0; j < STEPS; j++) {
        if (in->var_bytes == 2)
          GR_LAUNCH("incr_step_kernel", st, incr_step_kernel<int16_t><<<igrid, IT, hs, st>>>(
                                                in->bits, ld, in->m, U, counts, in->pos_off,
                                                (const int16_t *)in->pos_var, in->w, ctrl, wpicks));
        else
          GR_LAUNCH("incr_step_kernel", st, incr_step_kernel<int32_t><<<igrid, IT, hs, st>>>(
                                                in->bits, ld, in->m, U, counts, in->pos_off,
                                                (const int32_t *)in->pos_var, in->w, ctrl, wpicks));
      }
      GR_CUDA(cudaMemcpyAsync(h, ctrl, sizeof(GCtrl), cudaMemcpyDeviceToHost, st));
      GR_CUDA(cudaStreamSynchronize(st));
      if (((GCtrl *)h)->done) break;
      if ((long long)round * STEPS > (long long)in->m + 2 * STEPS) {
        gr_set_error("greedy did not terminate");
        return GR_ECUDA;
      }
    }
  }
  if (eager) {
    // pass t reads U[t & 1] and writes U[(t & 1) ^ 1]; parity is host-known
    // because every pass (even a no-op after done) flips it in argmax_kernel.
    for (;;) {
      for (int j = 0; j < CHUNK; j++, t++) {
        CountParams p{in->bits, ld, in->m, ntiles, U + (size_t)(t & 1) * ld,
                      U + (size_t)((t & 1) ^ 1) * ld, counts, ctrl, 1};
        GR_LAUNCH("count_kernel", (cudaStream_t)s, count_kernel<<<grid, CT, COUNT_SMEM_V2, st>>>(p));
        GR_LAUNCH("argmax_kernel", (cudaStream_t)s, argmax_kernel<<<1, AT, 0, st>>>(counts, in->m, in->w, ctrl, wpicks));
      }
      GR_CUDA(cudaMemcpyAsync(h, ctrl, sizeof(GCtrl), cudaMemcpyDeviceToHost, st));
      GR_CUDA(cudaStreamSynchronize(st));
      if (((GCtrl *)h)->done) break;
      if (t > 2 * in->m + 2 * CHUNK) { gr_set_error("greedy did not terminate"); return GR_ECUDA; }
    }
  }
  const int np = ((GCtrl *)h)->npicks;
  if (n_picks) *n_picks = np;
  // prune (reverse-delete, R12)
  GR_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * (in->m + 1), st));
  GR_LAUNCH("planes_build_kernel", (cudaStream_t)s, planes_build_kernel<<<(int)std::min<int64_t>((ld + 255) / 256, 148 * 8), 256, 0, st>>>(
      in->bits, ld, wpicks, ctrl, planes, L.nplanes));
  u64 *one = U;  // the U buffers are free once the greedy loop is done
  const int egrid = (int)std::min<int64_t>((ld + 255) / 256, 148 * 8);
  GR_LAUNCH("one_kernel", (cudaStream_t)s, one_kernel<<<egrid, 256, 0, st>>>(planes, L.nplanes, ld, one));
  GR_LAUNCH("private_kernel", (cudaStream_t)s, private_kernel<<<148 * 4, 256, 0, st>>>(in->bits, ld, wpicks, ctrl, one, flags, -1));
  std::vector<int> hflags(np + 1), hpicks(np + 1);
  if (np > 0) {
    GR_CUDA(cudaMemcpyAsync(hflags.data(), flags, sizeof(int) * np, cudaMemcpyDeviceToHost, st));
    GR_CUDA(cudaMemcpyAsync(hpicks.data(), wpicks, sizeof(int) * np, cudaMemcpyDeviceToHost, st));
    GR_CUDA(cudaStreamSynchronize(st));
  }
  // a pick that is the sole hitter of some clause stays so (counts only
  // decrease); the others are re-checked in removal order (R12): reverse pick
  // order, with weights descending weight and equal weights in reverse pick
  // order
  std::vector<int> removed(np + 1, 0);
  std::vector<int> ord;
  if ((rc = removal_order(in, hpicks, np, st, ord))) return rc;
  int *hf = pinned_ctrl() + 8;
  for (int j : ord) {
    if (hflags[j]) continue;
    GR_CUDA(cudaMemsetAsync(flags + j, 0, sizeof(int), st));
    GR_LAUNCH("private_kernel", (cudaStream_t)s, private_kernel<<<148 * 4, 256, 0, st>>>(in->bits, ld, wpicks, ctrl, one, flags, j));
    GR_CUDA(cudaMemcpyAsync(hf, flags + j, sizeof(int), cudaMemcpyDeviceToHost, st));
    GR_CUDA(cudaStreamSynchronize(st));
    if (!*hf) {
      removed[j] = 1;
      GR_LAUNCH("remove_kernel", (cudaStream_t)s, remove_kernel<<<egrid, 256, 0, st>>>(in->bits, ld, hpicks[j], planes, L.nplanes, one));
    }
  }
  // removed flags -> device (reuse `flags`)
  if (np > 0) {
    GR_CUDA(cudaMemcpyAsync(flags, removed.data(), sizeof(int) * np, cudaMemcpyHostToDevice, st));
    GR_CUDA(cudaStreamSynchronize(st));
  }
  GR_LAUNCH("finalize_kernel", (cudaStream_t)s, finalize_kernel<<<1, 256, 0, st>>>(wpicks, ctrl, flags, in->m, in->neg, in->n_neg, assign,
                                     status, smask));
  if (picks) GR_CUDA(cudaMemcpyAsync(picks, wpicks, sizeof(int) * in->m, cudaMemcpyDeviceToDevice, st));
  GR_CUDA(cudaStreamSynchronize(st));
  return GR_OK;
}

// ---- column-sharded greedy ------------------------------------
namespace {
struct ShardWS {
  GCtrl *ctrl;
  u64 *U, *planes, *smask;
  u32 *counts;
  int *picks, *flags;
  GLayout L;
};
int shard_ws(const gr_bitmatrix *in, void *ws, size_t ws_bytes, ShardWS &o) {
  int rc = validate_matrix(in);
  if (rc) return rc;
  o.L = glayout(in);
  if (!ws || ws_bytes < o.L.total) { gr_set_error("workspace too small"); return GR_EWORKSPACE; }
  char *base = (char *)ws;
  o.ctrl = (GCtrl *)(base + o.L.ctrl);
  o.U = (u64 *)(base + o.L.U);
  o.counts = (u32 *)(base + o.L.counts);
  o.picks = (int *)(base + o.L.picks);
  o.planes = (u64 *)(base + o.L.planes);
  o.flags = (int *)(base + o.L.flags);
  o.smask = (u64 *)(base + o.L.smask);
  return GR_OK;
}
bool shard_incremental(const gr_bitmatrix *in) {
  return in->pos_off != nullptr && in->pos_var != nullptr && in->m <= 50000 &&
         getenv("GR_GREEDY_EAGER") == nullptr;
}
}  // namespace

extern "C" size_t gr_greedy_shard_workspace_bytes(const gr_bitmatrix *shard) {
  return gr_greedy_matrix_workspace_bytes(shard);
}

extern "C" int gr_greedy_shard_begin(const gr_bitmatrix *shard, uint32_t *d_counts, void *ws,
                                     size_t ws_bytes, gr_stream_t s) {
  ShardWS w;
  int rc = shard_ws(shard, ws, ws_bytes, w);
  if (rc) return rc;
  if (!d_counts) { gr_set_error("null counts"); return GR_EINVAL; }
  cudaStream_t st = (cudaStream_t)s;
  const int64_t ld = shard->ld;
  GR_LAUNCH("init_kernel", st, init_kernel<<<592, 256, 0, st>>>(w.U, ld, shard->n_pos, w.ctrl, w.counts, shard->m, w.picks));
  count_grid();
  if (shard_incremental(shard)) {
    const int hgrid = (int)std::min<int64_t>((shard->n_pos * 9 + 255) / 256, 148 * 8);
    const size_t hs = sizeof(u32) * (size_t)shard->m;
    if (shard->var_bytes == 2)
      GR_LAUNCH("csr_hist_kernel", st, csr_hist_kernel<int16_t><<<std::max(hgrid, 1), 256, hs, st>>>(
                                          shard->n_pos, shard->pos_off, (const int16_t *)shard->pos_var, shard->m, w.counts));
    else
      GR_LAUNCH("csr_hist_kernel", st, csr_hist_kernel<int32_t><<<std::max(hgrid, 1), 256, hs, st>>>(
                                          shard->n_pos, shard->pos_off, (const int32_t *)shard->pos_var, shard->m, w.counts));
  } else {
    CountParams p{shard->bits, ld, shard->m, (int)((ld + TW - 1) / TW), w.U, nullptr, w.counts,
                  nullptr, 0};
    GR_LAUNCH("count_kernel", st, count_kernel<<<count_grid(), CT, COUNT_SMEM_V2, st>>>(p));
  }
  GR_CUDA(cudaMemcpyAsync(d_counts, w.counts, sizeof(u32) * shard->m, cudaMemcpyDeviceToDevice, st));
  return GR_OK;
}

extern "C" int gr_greedy_shard_step(const gr_bitmatrix *shard, uint32_t *d_counts, void *ws,
                                    size_t ws_bytes, gr_stream_t s) {
  ShardWS w;
  int rc = shard_ws(shard, ws, ws_bytes, w);
  if (rc) return rc;
  if (!d_counts) { gr_set_error("null counts"); return GR_EINVAL; }
  cudaStream_t st = (cudaStream_t)s;
  const int64_t ld = shard->ld;
  const bool inc = shard_incremental(shard);
  GR_LAUNCH("shard_pick_kernel", st, shard_pick_kernel<<<1, IT, 0, st>>>(d_counts, shard->m, shard->w, w.ctrl, w.picks, w.counts, inc ? 0 : 1));
  if (inc) {
    const size_t hs = sizeof(u32) * (size_t)shard->m;
    if (shard->var_bytes == 2)
      GR_LAUNCH("incr_step_kernel", st, (incr_step_kernel<int16_t, false><<<count_grid(), IT, hs, st>>>(
                                            shard->bits, ld, shard->m, w.U, w.counts, shard->pos_off,
                                            (const int16_t *)shard->pos_var, shard->w, w.ctrl, w.picks)));
    else
      GR_LAUNCH("incr_step_kernel", st, (incr_step_kernel<int32_t, false><<<count_grid(), IT, hs, st>>>(
                                            shard->bits, ld, shard->m, w.U, w.counts, shard->pos_off,
                                            (const int32_t *)shard->pos_var, shard->w, w.ctrl, w.picks)));
  } else {
    const int egrid = (int)std::min<int64_t>((ld + 255) / 256, 148 * 8);
    GR_LAUNCH("shard_mark_kernel", st, shard_mark_kernel<<<egrid, 256, 0, st>>>(shard->bits, ld, w.U, w.ctrl));
    CountParams p{shard->bits, ld, shard->m, (int)((ld + TW - 1) / TW), w.U, nullptr, w.counts,
                  w.ctrl, 0};
    GR_LAUNCH("count_kernel", st, count_kernel<<<count_grid(), CT, COUNT_SMEM_V2, st>>>(p));
  }
  GR_CUDA(cudaMemcpyAsync(d_counts, w.counts, sizeof(u32) * shard->m, cudaMemcpyDeviceToDevice, st));
  return GR_OK;
}

extern "C" int gr_greedy_shard_state(const gr_bitmatrix *shard, const void *ws, size_t ws_bytes,
                                     int32_t *n_picks, int32_t *done, int32_t *d_picks,
                                     gr_stream_t s) {
  ShardWS w;
  int rc = shard_ws(shard, (void *)ws, ws_bytes, w);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)s;
  int *h = pinned_ctrl();
  if (!h) { gr_set_error("cudaMallocHost failed"); return GR_ECUDA; }
  GR_CUDA(cudaMemcpyAsync(h, w.ctrl, sizeof(GCtrl), cudaMemcpyDeviceToHost, st));
  if (d_picks)
    GR_CUDA(cudaMemcpyAsync(d_picks, w.picks, sizeof(int) * shard->m, cudaMemcpyDeviceToDevice, st));
  GR_CUDA(cudaStreamSynchronize(st));
  if (n_picks) *n_picks = ((GCtrl *)h)->npicks;
  if (done) *done = ((GCtrl *)h)->done;
  return GR_OK;
}

extern "C" int gr_greedy_shard_private(const gr_bitmatrix *shard, int32_t only, int32_t *d_flags,
                                       void *ws, size_t ws_bytes, gr_stream_t s) {
  ShardWS w;
  int rc = shard_ws(shard, ws, ws_bytes, w);
  if (rc) return rc;
  if (!d_flags) { gr_set_error("null flags"); return GR_EINVAL; }
  cudaStream_t st = (cudaStream_t)s;
  const int64_t ld = shard->ld;
  const int egrid = (int)std::min<int64_t>((ld + 255) / 256, 148 * 8);
  u64 *one = w.U + ld;  // the second U buffer is free after the greedy loop
  if (only < 0) {
    GR_LAUNCH("planes_build_kernel", st, planes_build_kernel<<<egrid, 256, 0, st>>>(shard->bits, ld, w.picks, w.ctrl, w.planes, w.L.nplanes));
    GR_LAUNCH("one_kernel", st, one_kernel<<<egrid, 256, 0, st>>>(w.planes, w.L.nplanes, ld, one));
  }
  GR_LAUNCH("private_kernel", st, private_kernel<<<148 * 4, 256, 0, st>>>(shard->bits, ld, w.picks, w.ctrl, one, d_flags, only));
  return GR_OK;
}

extern "C" int gr_greedy_shard_remove(const gr_bitmatrix *shard, int32_t j, void *ws,
                                      size_t ws_bytes, gr_stream_t s) {
  ShardWS w;
  int rc = shard_ws(shard, ws, ws_bytes, w);
  if (rc) return rc;
  if (j < 0 || j >= shard->m) { gr_set_error("pick index out of range"); return GR_EINVAL; }
  cudaStream_t st = (cudaStream_t)s;
  const int64_t ld = shard->ld;
  const int egrid = (int)std::min<int64_t>((ld + 255) / 256, 148 * 8);
  int v = -1;
  GR_CUDA(cudaMemcpyAsync(&v, w.picks + j, sizeof(int), cudaMemcpyDeviceToHost, st));
  GR_CUDA(cudaStreamSynchronize(st));
  if (v < 0 || v >= shard->m) { gr_set_error("no such pick"); return GR_EINVAL; }
  GR_LAUNCH("remove_kernel", st, remove_kernel<<<egrid, 256, 0, st>>>(shard->bits, ld, v, w.planes, w.L.nplanes, w.U + ld));
  return GR_OK;
}

extern "C" int gr_greedy_shard_finalize(const gr_bitmatrix *shard, const int32_t *d_removed,
                                        uint64_t *assign, int32_t *status, void *ws,
                                        size_t ws_bytes, gr_stream_t s) {
  ShardWS w;
  int rc = shard_ws(shard, ws, ws_bytes, w);
  if (rc) return rc;
  if (!d_removed || !assign || !status) { gr_set_error("null removed / assign / status"); return GR_EINVAL; }
  cudaStream_t st = (cudaStream_t)s;
  GR_LAUNCH("finalize_kernel", st, finalize_kernel<<<1, 256, 0, st>>>(w.picks, w.ctrl, d_removed, shard->m, shard->neg, shard->n_neg, assign, status, w.smask));
  return GR_OK;
}
