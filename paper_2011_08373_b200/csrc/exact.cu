// exact.cu -- exact PMS / WPMS (gr_solve_pms) and exact MHS (gr_mhs_exact).
//
// Method (PAPER.md:15 PMS/WPMS, PAPER.md:11 MHS, PAPER.md:24 MaxSAT
// strategy): minimise the (weighted) number of true b_i subject to phi.  The
// canonical optimum is the smallest colex rank at the optimal level (reading
// R2) or the minimum (W, k, rank) key (reading R3).
//
// B200 design:
//   pack_kernel     one CTA per instance: validation (R4, R6, R8), support
//                   restriction + order-preserving relabel (R13), dedup and
//                   subsumption, ascending-size clause order, sorted-weight
//                   prefix sums S_k.
//   enum_kernel     persistent CTAs (grid = SMs x occupancy) pull fixed-size
//                   chunks of the current level's colex rank range from a
//                   global atomic counter; each lane walks a contiguous
//                   sub-range.  A candidate is x = U | S with S its J =
//                   min(k, JMAX) lowest elements; the walk visits sub-blocks
//                   (fixed U, S ranging over the j-subsets of a small region
//                   [0, R_j), at most 128 candidates = one two-word mask F) in
//                   rank order.  A positive clause P that U misses narrows F by
//                   its precomputed record H_j(P); a negative clause with at
//                   most j variables outside U removes the S that hold them
//                   all.  Clause records are staged in shared memory
//                   (broadcast reads).  Canonical minimum: per-lane first
//                   witness -> warp shuffle-min -> CTA min -> one 64-bit
//                   atomicMin per chunk.
//   finish_kernel   one CTA: commits level k for every active instance
//                   (decode, weighted incumbent, S_k stop rule, k_max), writes
//                   finished results, compacts the active list and plans the
//                   chunk ranges of level k+1 (block scan).
#include <cub/block/block_scan.cuh>

#include <algorithm>
#include <cstddef>
#include <atomic>
#include <cstdlib>
#include <mutex>

#include "common.cuh"

namespace {

constexpr int NT = 256;          // enumeration CTA size
#ifndef GR_FT
#define GR_FT 1024
#endif
constexpr int FT = GR_FT;        // finish CTA size
constexpr int PT = 128;          // pack CTA size
constexpr int MAXC = 4096;       // max clauses per instance (exact solvers)

struct Ctrl {
  u64 next_chunk;     // atomic chunk counter of the running level
  u64 total_chunks;   // chunks of the running level
  int n_active;       // instances listed for the running level
  int n_remaining;    // instances not finished (listed or waiting for their start level)
  u64 lane_cands;     // candidates per lane per chunk (L)
  unsigned fin_ticket;  // finish: blocks done committing (the last one plans)
  unsigned pad0;
  // the level loop on the device (queue_kernel)
  u64 q_tickets;        // tickets handed out: a CTA takes ticket e and works the task of ring entry e
  u64 q_entries;        // ring entries allocated by enqueuers
  long long q_budget;   // ring entries available beyond one per open instance
  u64 q_tasks;          // task records allocated
  int q_remaining;      // open (instance, solve) units; 0 ends the launch
  int pad2;
  u64 q_work;           // candidates of the published, uncommitted tasks (lane window sizing)
  u64 pad3[5];
};
static_assert(sizeof(Ctrl) == 128, "Ctrl layout");

// Level k of instance b of solve sv: one task record, worked by every CTA
// whose ticket maps to one of its ring entries.  A task may be
// speculative: level k+1 published while level k still runs; it commits only
// after level k confirmed it, and is cancelled if level k ends the instance.
constexpr unsigned SUCC_CLOSED = 0xffffffffu;
struct Task {
  u64 claimed;   // warp chunks handed out (atomic)
  u64 pending;   // warp chunks not finished, + 1 while unconfirmed; the decrement to 0 commits
  u64 nchunks;   // warp chunks of the level: 32 lane windows of L candidates each
  u64 L;         // lane window
  i64 key[2];    // the level's minimum keys (fused: PMS, MHS)
  int b, k;
  unsigned succ;  // 0: no successor yet; SUCC_CLOSED: none may attach; else successor index + 1
  unsigned char sv, rb, depth, cancelled;  // solve; weighted key shift; speculation depth
                                           // (0 = confirmed); cancelled speculation
  u64 t_make, t_exhaust, t_commit, t_unused;  // globaltimer (ns): the level timeline
                                              // (scripts/queue_stats.py)
  u64 pad[4];
};
static_assert(sizeof(Task) == 128, "Task layout");
// A ring entry is one u64: generation (12 bits) | ring round of its ticket
// (12 bits) | extra-entry flag | solve | task record index (38 bits); the
// waiter of ticket e knows the generation and e's round, so a stale entry of
// an earlier launch or round never matches.
typedef u64 RingEntry;
constexpr int QLEVELS = 132;  // task records per (instance, solve): two per level (speculation)
// ring entries: a power of two above one entry per open unit of two solves
// plus the tickets the grid can hold
__host__ __device__ inline u64 ring_cap(int B) {
  u64 need = 8ull * (u64)B + 16384ull, c = 65536;
  while (c < need) c <<= 1;
  return c;
}

#ifndef GR_JMAX
#define GR_JMAX 13
#endif
constexpr int JMAX = GR_JMAX;  // S = the J = min(k, JMAX) lowest elements of a candidate
static_assert(JMAX >= 2 && JMAX <= 14, "the iterator's ancestor stack holds J - 2 entries");
constexpr int HREC = JMAX - 1;  // per-clause records H_2, ..., H_JMAX (H_1(P) = P itself)
constexpr int HX = 16;         // HIT_j({x}) is 0 for x >= R_j, and R_j <= 16 for j >= 2

struct Layout {
  size_t ctrl, meff, npr, nnr, kmax, ks, done, rb, sup, decided, bestx, bestw, wtot, lvlkey, sk, wr,
      active, chunk_base, pk, hrec, ptmp, tasks, ring, gcost, total;
};

Layout layout_of(const gr_batch *in) {
  Layout L{};
  size_t B = (size_t)in->B, o = 0;
  auto take = [&](size_t bytes) { size_t at = o; o = align256(o + bytes); return at; };
  L.ctrl = take(sizeof(Ctrl));
  L.meff = take(4 * B);
  L.npr = take(4 * B);
  L.nnr = take(4 * B);
  L.kmax = take(4 * B);
  L.ks = take(4 * B);
  L.done = take(4 * B);
  L.rb = take(4 * B);
  L.sup = take(16 * B);
  L.decided = take(8 * B);
  L.bestx = take(8 * B);
  L.bestw = take(8 * B);
  L.wtot = take(8 * B);
  L.lvlkey = take(8 * B);
  L.sk = take(8 * 65 * B);
  L.wr = take(4 * 64 * B);
  L.active = take(4 * 2 * B);
  L.chunk_base = take(8 * (B + 1));
  L.ptmp = take(8 * B);
  L.pk = take(8 * (size_t)std::max<int64_t>(in->total_clauses, 1));
  L.hrec = take(16 * HREC * (size_t)std::max<int64_t>(in->total_clauses, 1));
  L.tasks = take(sizeof(Task) * QLEVELS * B);
  L.ring = take(sizeof(RingEntry) * ring_cap(in->B));
  L.gcost = take(8 * B);  // gr_solve(GR_STRATEGY_MHS_FINAL): the greedy answers' costs
  L.total = o;
  return L;
}

struct WS {
  Ctrl *ctrl;
  int *meff, *npr, *nnr, *kmax, *ks, *done, *rb;
  u64 *sup, *decided, *bestx, *bestw, *wtot;
  i64 *lvlkey;
  u64 *sk;
  u32 *wr;
  int *active;
  u64 *chunk_base;
  u64 *ptmp;       // finish scratch: level size per listed position (~0: not listed)
  u64 *pk, *hrec;  // packed clause masks; [clause][HREC] two-word H_j(P) records of the positives
  Task *tasks;     // queue_kernel: task records of this solve
  RingEntry *ring; // queue_kernel: the ticket ring (the first solve's)
};

WS ws_of(const gr_batch *in, void *base) {
  Layout L = layout_of(in);
  char *p = (char *)base;
  WS w;
  w.ctrl = (Ctrl *)(p + L.ctrl);
  w.meff = (int *)(p + L.meff);
  w.npr = (int *)(p + L.npr);
  w.nnr = (int *)(p + L.nnr);
  w.kmax = (int *)(p + L.kmax);
  w.ks = (int *)(p + L.ks);
  w.done = (int *)(p + L.done);
  w.rb = (int *)(p + L.rb);
  w.sup = (u64 *)(p + L.sup);
  w.decided = (u64 *)(p + L.decided);
  w.bestx = (u64 *)(p + L.bestx);
  w.bestw = (u64 *)(p + L.bestw);
  w.wtot = (u64 *)(p + L.wtot);
  w.lvlkey = (i64 *)(p + L.lvlkey);
  w.sk = (u64 *)(p + L.sk);
  w.wr = (u32 *)(p + L.wr);
  w.active = (int *)(p + L.active);
  w.chunk_base = (u64 *)(p + L.chunk_base);
  w.ptmp = (u64 *)(p + L.ptmp);
  w.pk = (u64 *)(p + L.pk);
  w.hrec = (u64 *)(p + L.hrec);
  w.tasks = (Task *)(p + L.tasks);
  w.ring = (RingEntry *)(p + L.ring);
  return w;
}

struct In {
  int B, W, max_clauses, wstride;
  const int32_t *m;
  const int64_t *off;
  const int32_t *n_pos;
  const uint64_t *masks;
  const uint32_t *w;
  const int32_t *sel;  // optional: solve only instances with sel[b] == sel_val (others untouched)
  int sel_val;
  const int32_t *kstart;  // optional (unit weights): first level to enumerate (f2)
};
struct Out {
  uint64_t *assign, *cost, *decided;
  int32_t *status;
};

thread_local const int32_t *t_sel = nullptr;  // set by gr_solve around its fallback solve
thread_local int t_sel_val = 0;

In in_of(const gr_batch *b, int which) {
  const bool unit = which != 0 || b->w == nullptr;
  In r{b->B, b->W, b->max_clauses, b->wstride, b->m, b->off, b->n_pos, b->masks,
       which == 0 ? b->w : nullptr, t_sel, t_sel_val, unit ? b->k_start : nullptr};
  return r;
}
Out out_of(const gr_result *o) { return Out{o->assign, o->cost, o->decided, o->status}; }

// ---------------------------------------------------------------------------
// finalisation of one instance (single thread)
// ---------------------------------------------------------------------------
__device__ void write_result(const In &in, const Out &out, int b, int status, u64 x_rel, u64 s0,
                             u64 s1, u64 cost, u64 decided, int which) {
  u64 a0 = 0, a1 = 0;
  if (status == GR_SAT) {
    pdep128(x_rel, s0, s1, a0, a1);
    if (which == 1) {  // MHS: flag phi- 
      int64_t lo = in.off[b], hi = in.off[b + 1];
      for (int64_t j = lo + in.n_pos[b]; j < hi; j++) {
        u64 n0 = in.masks[j * in.W], n1 = in.W > 1 ? in.masks[j * in.W + 1] : 0;
        if ((a0 & n0) == n0 && (a1 & n1) == n1) { status = GR_SAT_NEG_VIOLATED; break; }
      }
    }
  } else {
    cost = ~0ull;
  }
  out.assign[(size_t)b * in.W] = a0;
  if (in.W > 1) out.assign[(size_t)b * in.W + 1] = a1;
  out.cost[b] = cost;
  out.status[b] = status;
  if (out.decided) out.decided[b] = decided;
}

// A sub-block's candidate mask: up to 128 candidates in two words.
struct F2 {
  u64 lo, hi;
};
__device__ F2 hitting(int j, u64 p);

// ---------------------------------------------------------------------------
// pack: one CTA per instance
// ---------------------------------------------------------------------------
// one pack launch packs one batch for up to two solves (the PMS and the MHS
// workspaces of gr_solve_pms_mhs): CTA i < in0.B packs instance i for
// (in0, ws0), CTA in0.B + i for (in1, ws1); the first CTA of each solve also
// resets its control block (lane_cands = the fixed window, 0 = adaptive)
struct PackArgs {
  In in[2];
  Out out[2];
  WS ws[2];
  int which[2];
  u64 lane_cands;
  u64 ring_n;  // entries of ws[0]'s ticket ring, cleared by the pack's CTAs
};
__device__ void pack_body(const In &in, const Out &out, const WS &ws, int which, int b);
__global__ void __launch_bounds__(PT) pack_kernel(const __grid_constant__ PackArgs A) {
  const int s = (int)blockIdx.x >= A.in[0].B ? 1 : 0;
  const int b = (int)blockIdx.x - (s ? A.in[0].B : 0);
  if (b == 0 && threadIdx.x < sizeof(Ctrl) / 8) {
    u64 *c = (u64 *)A.ws[s].ctrl;
    c[threadIdx.x] = threadIdx.x == offsetof(Ctrl, lane_cands) / 8 ? A.lane_cands : 0ull;
  }
  {  // clear a slice of the ring: no entry of an earlier launch (e.g. a CUDA
     // graph replay, whose launch generation is fixed) can match a ticket
    const u64 g = gridDim.x, i = blockIdx.x;
    for (u64 q = A.ring_n * i / g + threadIdx.x; q < A.ring_n * (i + 1) / g; q += blockDim.x) A.ws[0].ring[q] = 0ull;
  }
  pack_body(A.in[s], A.out[s], A.ws[s], A.which[s], b);
}
__device__ void pack_body(const In &in, const Out &out, const WS &ws, int which, int b) {
  extern __shared__ u64 sm[];  // [max_clauses] masks, [max_clauses] int info, [max_clauses] u8 keep
  __shared__ int s_bad, s_unsat, s_negempty, s_npr, s_nnr;
  __shared__ unsigned long long s_sup0, s_sup1;
  __shared__ u32 s_w[64];
  __shared__ u64 s_ws[64];
  const int t = threadIdx.x;
  if (in.sel && in.sel[b] != in.sel_val) {  // not selected: leave its results alone
    if (t == 0) ws.done[b] = 1;
    return;
  }
  u64 *R = sm;
  int *info = (int *)(sm + in.max_clauses);
  unsigned char *keep0 = (unsigned char *)(info + in.max_clauses);
  const int64_t lo = in.off[b], n64 = in.off[b + 1] - lo;
  const int m = in.m[b], np = in.n_pos[b], W = in.W;
  if (t == 0) {
    s_bad = (n64 < 0 || n64 > in.max_clauses || np < 0 || np > n64 || m < 0 || m > 64 * W);
    s_unsat = 0;
    s_negempty = 0;
    s_sup0 = 0;
    s_sup1 = 0;
    s_npr = 0;
    s_nnr = 0;
  }
  __syncthreads();
  const int n = s_bad ? 0 : (int)n64;
  // validation (R8 bits >= m, R6 empty clause) and support of phi+
  const u64 al0 = m >= 64 ? ~0ull : ((1ull << m) - 1);
  const u64 al1 = m >= 128 ? ~0ull : (m <= 64 ? 0ull : ((1ull << (m - 64)) - 1));
  u64 sup0 = 0, sup1 = 0;
  for (int j = t; j < n; j += PT) {
    u64 x0 = in.masks[(lo + j) * W], x1 = W > 1 ? in.masks[(lo + j) * W + 1] : 0;
    if ((x0 & ~al0) | (x1 & ~al1)) s_bad = 1;
    if (!(x0 | x1)) {
      if (j < np) s_unsat = 1;
      else s_negempty = 1;
    }
    if (j < np) { sup0 |= x0; sup1 |= x1; }
  }
  if (in.w)
    for (int i = t; i < m; i += PT)
      if (in.w[(size_t)b * in.wstride + i] == 0) s_bad = 1;
  if (sup0) atomicOr(&s_sup0, (unsigned long long)sup0);
  if (sup1) atomicOr(&s_sup1, (unsigned long long)sup1);
  __syncthreads();
  sup0 = s_sup0;
  sup1 = s_sup1;
  const int me = __popcll(sup0) + __popcll(sup1);
  int status = -1;
  if (s_bad) status = GR_BADINPUT;
  else if (s_unsat || (which == 0 && s_negempty)) status = GR_UNSAT;
  else if (me > 64) status = GR_UNSUPPORTED;
  // an empty negative clause decides the PMS (UNSAT) but not the MHS: the
  // clauses are still packed, for a fused PMS + MHS walk (gr_solve_pms_mhs)
  const bool decided_here = status >= 0;
  if (decided_here) {
    if (t == 0) {
      ws.done[b] = 1;
      write_result(in, out, b, status, 0, 0, 0, 0, 0, which);
    }
    if (!(status == GR_UNSAT && !s_unsat)) return;
  }
  // relabel onto the support; negatives that touch a non-support variable are
  // always satisfied by an optimum (those variables are false) -> dropped (R13)
  const int nneg_in = which == 0 ? n - np : 0;
  const int nc = np + nneg_in;
  for (int j = t; j < nc; j += PT) {
    u64 x0 = in.masks[(lo + j) * W], x1 = W > 1 ? in.masks[(lo + j) * W + 1] : 0;
    int keep = 1;
    if (j >= np && ((x0 & ~sup0) | (x1 & ~sup1))) keep = 0;
    R[j] = keep ? pext128(x0, x1, sup0, sup1) : 0;
    keep0[j] = (unsigned char)keep;
  }
  __syncthreads();
  // dedup + subsumption within each polarity: drop j if another kept clause i
  // of the same polarity has R[i] subset of R[j] (and R[i] != R[j] or i < j).
  // The feasible set is unchanged (a hitting set of R[i] hits R[j]; an
  // assignment avoiding all of N_i avoids N_j, N_i subset of N_j).
  for (int j = t; j < nc; j += PT) {
    int keep = keep0[j];
    if (keep) {
      const int a0 = j < np ? 0 : np, a1 = j < np ? np : nc;
      const u64 rj = R[j];
      for (int i = a0; i < a1; i++) {
        if (i == j || !keep0[i]) continue;
        const u64 ri = R[i];
        if ((ri & ~rj) == 0 && (ri != rj || i < j)) { keep = 0; break; }
      }
    }
    info[j] = keep ? (1 | (__popcll(R[j]) << 8)) : 0;
    if (keep) atomicAdd(j < np ? &s_npr : &s_nnr, 1);
  }
  __syncthreads();
  const int npr = s_npr;
  // ascending clause size, stable by index, positives first: destination =
  // number of kept clauses of the same polarity ordered before j
  for (int j = t; j < nc; j += PT) {
    const int ij = info[j];
    if (!ij) continue;
    const int a0 = j < np ? 0 : np, a1 = j < np ? np : nc;
    const int pj = ij >> 8;
    int d = 0;
    for (int i = a0; i < a1; i++) {
      const int ii = info[i];
      if (!ii) continue;
      const int pi = ii >> 8;
      d += (pi < pj || (pi == pj && i < j));
    }
    const int64_t dst = lo + (j < np ? 0 : npr) + d;
    ws.pk[dst] = R[j];
    if (j < np)
      for (int jj = 2; jj <= JMAX; jj++) ((F2 *)ws.hrec)[dst * HREC + jj - 2] = hitting(jj, R[j]);
  }
  // weights of the support variables (relabelled order) and S_k
  if (t < 64) {
    u32 wv = 0;
    if (t < me) {
      // original index of the t-th support variable
      u64 s0 = sup0, s1 = sup1;
      int idx = -1;
      for (int q = 0; q <= t; q++) {
        if (s0) { u64 l = s0 & (~s0 + 1); idx = __ffsll((long long)l) - 1; s0 ^= l; }
        else { u64 l = s1 & (~s1 + 1); idx = 64 + __ffsll((long long)l) - 1; s1 ^= l; }
      }
      wv = in.w ? in.w[(size_t)b * in.wstride + idx] : 1u;
    }
    s_w[t] = wv;
    ws.wr[(size_t)b * 64 + t] = wv;
  }
  __syncthreads();
  if (t < me) {  // rank of weight t among the support weights (ties by index)
    u32 wt = s_w[t];
    int r = 0;
    for (int i = 0; i < me; i++) r += (s_w[i] < wt) || (s_w[i] == wt && i < t);
    s_ws[r] = wt;
  }
  __syncthreads();
  if (t == 0) {
    const int nnr = s_nnr;
    u64 *sk = ws.sk + (size_t)b * 65;
    u64 acc = 0;
    sk[0] = 0;
    for (int i = 0; i < 64; i++) {
      if (i < me) acc += s_ws[i];
      sk[i + 1] = acc;
    }
    ws.meff[b] = me;
    ws.npr[b] = npr;
    ws.nnr[b] = nnr;
    ws.kmax[b] = me < npr ? me : npr;
    // f2: the caller guarantees no feasible set below k_start[b] (e.g. the
    // previous optimum level of a sub-formula): those levels are skipped
    const int ks = in.kstart ? (in.kstart[b] > 1 ? in.kstart[b] : 1) : 1;
    ws.ks[b] = ks;
    ws.sup[2 * b] = sup0;
    ws.sup[2 * b + 1] = sup1;
    ws.wtot[b] = acc;
    ws.bestw[b] = ~0ull;
    ws.bestx[b] = 0;
    ws.lvlkey[b] = GR_KEY_NONE;
    ws.decided[b] = 1;  // level 0: the empty assignment
    if (decided_here) {
      // done at pack (see above); the packed clauses serve a fused MHS only
    } else if (npr == 0) {
      // phi+ empty: the all-false assignment satisfies every (non-empty)
      // negative clause and is optimal
      ws.done[b] = 1;
      write_result(in, out, b, GR_SAT, 0, sup0, sup1, 0, 1, which);
    } else if (ks > (me < npr ? me : npr)) {  // nothing left to enumerate (R13)
      ws.done[b] = 1;
      write_result(in, out, b, GR_UNSAT, 0, sup0, sup1, 0, 1, which);
    } else {
      ws.done[b] = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// the level walk of one lane: bit-parallel decision of the J lowest elements
// ---------------------------------------------------------------------------
// Candidates at level k are k-subsets x of [0, m_eff) in colex order (rank =
// sum_i C(c_i, i)).  With J = min(JMAX, k), split x = U | S, S = the J lowest
// elements.  All candidates sharing U form one contiguous rank block, S
// ranging over the J-subsets of [0, min U) in colex order.  Recursively,
//   node(j, U, e, base) = part A: the j-subsets of [0, min(e, R_j))   (one
//                                 sub-block, <= 128 candidates)
//                         part B: for t in [R_j, e): node(j-1, U | {t}, t,
//                                 base + C(t, j))
// where R_j is the largest R with C(R, j) <= 128 (R = 64, 16, 10, 9, 9, 9, 10,
// 10, 11, 12 for j = 1..10).  A sub-block's candidates are the bits of one
// two-word mask F whose bit index is the colex offset idx_j(S) = sum_i
// C(s_i, i), so rank = base + bit.  A positive clause P missed by U keeps the candidates
// that meet P: F &= H_j(P), H_j(P) = {j-subsets of [0, R_j) meeting P}
// (precomputed per clause by the pack; H_1(P) = P).  A negative clause N
// whose variables outside the region all lie in U kills the S that contain
// N's region part.  Each lane visits one sub-block per loop iteration (a flat
// depth-first iterator over the node tree), so the lanes of a warp run the
// same clause-test code in lock step.  An inner node's whole subtree is
// first checked for a refutation by one clause scan (refuted_by).


__device__ __forceinline__ F2 f2_and(F2 a, F2 b) { return F2{a.lo & b.lo, a.hi & b.hi}; }
__device__ __forceinline__ F2 f2_andnot(F2 a, F2 b) { return F2{a.lo & ~b.lo, a.hi & ~b.hi}; }
__device__ __forceinline__ bool f2_any(F2 a) { return (a.lo | a.hi) != 0; }
__device__ __forceinline__ F2 f2_nbits(u64 n) {  // the n lowest bits, n <= 128
  return n >= 128 ? F2{~0ull, ~0ull}
                  : (n >= 64 ? F2{~0ull, (1ull << (n - 64)) - 1ull} : F2{(1ull << n) - 1ull, 0ull});
}
__device__ __forceinline__ int f2_ctz(F2 a) {
  return a.lo ? __ffsll((long long)a.lo) - 1 : 64 + __ffsll((long long)a.hi) - 1;
}
__device__ __forceinline__ int f2_popc(F2 a) { return __popcll(a.lo) + __popcll(a.hi); }

// R_j = the largest region with C(R_j, j) <= 128 (j = 1: every variable)
__host__ __device__ constexpr int region_of(int j) {
  return j <= 8 ? (int)((0x0A0A0909090A1040ull >> (8 * (j - 1))) & 0xffull)  // 64 16 10 9 9 9 10 10
                : (j == 9 ? 11 : (j == 10 ? 12 : (j == 11 ? 13 : (j == 12 ? 14 : (j == 13 ? 15 : 16)))));
}
__device__ __forceinline__ u64 nbits(u64 n) { return n >= 64 ? ~0ull : ((1ull << n) - 1ull); }

// HIT_j({x}) for j <= JMAX, x < 64 (0 when x >= R_j), built at compile time:
// bit i set iff the i-th j-subset of [0, R_j) in colex order contains x.
struct HitTable {
  u64 lo[(JMAX + 1) * 64], hi[(JMAX + 1) * 64];
  constexpr HitTable() : lo(), hi() {
    for (int v = 0; v < 64; v++) lo[64 + v] = 1ull << v;  // j = 1: R_1 = 64, HIT = {x}
    for (int j = 2; j <= JMAX; j++) {
      const int R = region_of(j);
      u64 x = (1ull << j) - 1;
      for (int i = 0; x < (1ull << R); i++) {  // j-subsets of [0, R) in colex order
        for (int v = 0; v < R; v++)
          if (x >> v & 1ull) {
            if (i < 64) lo[64 * j + v] |= 1ull << i; else hi[64 * j + v] |= 1ull << (i - 64);
          }
        u64 c = x & (~x + 1), y = x + c;  // Gosper: next j-subset
        int tz = 0;
        while (!(c >> tz & 1ull)) tz++;
        x = y | (((y ^ x) >> 2) >> tz);
      }
    }
  }
};
static __device__ const HitTable g_hit = HitTable();

// H_j(p): bit i set iff the i-th j-subset of [0, R_j) (colex order) meets p,
// i.e. the union of HIT_j({x}) over the elements x of p
__device__ F2 hitting(int j, u64 p) {
  if (j == 1) return F2{p, 0ull};  // H_1(P) = P
  F2 r{0ull, 0ull};
  p &= nbits((u64)region_of(j));   // HIT_j({x}) = 0 for x >= R_j
  for (; p; p &= p - 1) {
    const int x = __ffsll((long long)p) - 1;
    r.lo |= g_hit.lo[64 * j + x];
    r.hi |= g_hit.hi[64 * j + x];
  }
  return r;
}

// Work counters of the counting instantiation (COUNT = true), the units of
// the exact solvers' roofline: positive / negative clause
// tests of a sub-block, clauses read by the subtree-refutation scans,
// sub-blocks tested, candidates in them, lane windows positioned (colex
// unrank).
struct Work {
  u64 pos = 0, neg = 0, scan = 0, blocks = 0, cands = 0, windows = 0;
};
enum { W_POS, W_NEG, W_SCAN, W_BLOCKS, W_CANDS, W_WINDOWS, W_WIDE, W_N = 8 };

extern __shared__ u64 g_dsmem[];  // dynamic shared memory of the enumeration kernels
__device__ __forceinline__ const F2 *tab_hitx() { return (const F2 *)g_dsmem; }
__device__ __forceinline__ const u64 *tab_cs() { return g_dsmem + 2 * (JMAX + 1) * HX; }
__device__ __forceinline__ const F2 *tab_lowb() { return (const F2 *)(tab_cs() + 65 * (JMAX + 1)); }
__device__ __forceinline__ const int *tab_reg() { return (const int *)(tab_lowb() + 129); }
__device__ __forceinline__ const unsigned char *tab_nb() { return (const unsigned char *)(tab_reg() + 16); }

template <typename M>
struct Clauses {
  const M *P;       // [np + nn] positives then negatives (uniform reads)
  const F2 *H;      // [np][HREC] H_j(P) at H[q * HREC + j - 1]
  // the tables at the start of dynamic shared memory (tab_*: fixed offsets
  // from one symbol, so the walk holds no pointer registers for them):
  //   HIT_j({x}) [JMAX + 1][HX], C(n, j) [65][JMAX + 1] for j <= JMAX, the n
  //   lowest bits [129], R_j [JMAX + 1], sub-block sizes C(min(e, R_j), j)
  int np, nn;
};

// Test one sub-block: F (its candidates in the lane's window) narrowed by
// every positive clause (test_pos), then by every negative clause (test_neg).
template <typename M, bool COUNT>
__device__ __forceinline__ F2 test_pos(int j, M U, F2 F, const Clauses<M> &c, Work &wk) {
  const int np = c.np;
  if (j == 1) {  // H_1(P) = P
    for (int q = 0; q < np; q++) {
      const M pq = c.P[q];
      if (!(U & pq)) F.lo &= (u64)pq;
      if (COUNT) wk.pos += 1;
      if (!(q & 3) && !F.lo) return F2{0ull, 0ull};
    }
    return F2{F.lo, 0ull};
  }
  const F2 *H = c.H + (j - 2);
  int q = 0;
  for (; q + 4 <= np; q += 4) {
    const M p0 = c.P[q], p1 = c.P[q + 1], p2 = c.P[q + 2], p3 = c.P[q + 3];
    const F2 h0 = H[HREC * q], h1 = H[HREC * (q + 1)], h2 = H[HREC * (q + 2)],
             h3 = H[HREC * (q + 3)];
    if (!(U & p0)) F = f2_and(F, h0);
    if (!(U & p1)) F = f2_and(F, h1);
    if (!(U & p2)) F = f2_and(F, h2);
    if (!(U & p3)) F = f2_and(F, h3);
    if (COUNT) wk.pos += 4;
    if (!f2_any(F)) return F;
  }
  for (; q < np; q++) {
    if (!(U & c.P[q])) F = f2_and(F, H[HREC * q]);
    if (COUNT) wk.pos += 1;
  }
  return F;
}

template <typename M, bool COUNT>
__device__ __forceinline__ F2 test_neg(int j, M U, int e, F2 F, const Clauses<M> &c, Work &wk) {
  const int np = c.np;
  const M lowm = (M)nbits((u64)e);
  const F2 *hx = tab_hitx() + HX * j;
  for (int t = 0; t < c.nn; t++) {
    M rest = c.P[np + t] & ~U;
    if (COUNT) wk.neg += 1;
    if ((rest & ~lowm) || popc(rest) > j) continue;  // some variable of N stays false
    F2 kill{~0ull, ~0ull};
    if (j == 1) {  // HIT_1({x}) = bit x
      if (rest) kill = F2{(u64)rest, 0ull};
    } else {
      for (; rest; rest &= rest - 1) kill = f2_and(kill, hx[ctz(rest)]);
    }
    F = f2_andnot(F, kill);  // the S holding every variable of N outside U
    if (!f2_any(F)) return F;
  }
  return F;
}

template <typename M, bool COUNT>
__device__ __forceinline__ F2 test_sub(int j, M U, int e, F2 F, const Clauses<M> &c, Work &wk) {
  F = test_pos<M, COUNT>(j, U, F, c, wk);
  if (!f2_any(F)) return F;
  return test_neg<M, COUNT>(j, U, e, F, c, wk);
}

// weighted: the weights of the j low elements encoded by bit idx (colex
// unrank of idx within [0, ea), downward scan over the shared binomials)
__device__ __forceinline__ u64 weight_low(int j, u64 idx, int ea, const u32 *w, const u64 *cs) {
  u64 W = 0;
  int c = ea - 1;
  for (int i = j; i >= 1; i--) {
    u64 v;
    while ((v = cs[c * (JMAX + 1) + i]) > idx) c--;
    W += w[c];
    idx -= v;
    c--;
  }
  return W;
}

// walk ranks [r_lo, r_lo + cnt) of level k.  MODE 0: unit weights, first
// witness; 1: unit, exhaustive; 2: weighted (min key W << rb | rank).
// Iterator state: the top-level U (k - J elements) with its first rank
// base_top, the path t_0 > t_1 > ... of part-B choices below it (6 bits
// each in tp), the current U and the current sub-block's first rank base.
// Is the whole subtree of node (j, U, e) -- every x = U | S, S a j-subset of
// [0, e) -- infeasible?  A positive clause missing U and [0, e), more than j
// pairwise disjoint positive clauses missing U (restricted to [0, e), greedy
// packing in clause order: S needs one element of each), or a negative
// clause inside U.
// 0: not refuted; 1: refuted by the positive clauses (for the MHS too);
// 2: only by a negative clause inside U
template <typename M, bool COUNT>
__device__ __forceinline__ int refuted_by(int j, M U, int e, const Clauses<M> &c, Work &wk) {
  const M lowe = (M)nbits((u64)e);
  M used = 0;
  int pk = 0, r = 0;
  bool dead = false;
  for (; r < c.np; r++) {
    const M pr = c.P[r];
    if (pr & U) continue;
    const M q = pr & lowe;
    if (!q) { dead = true; break; }
    if (!(q & used)) {
      used |= q;
      if (++pk > j) { dead = true; break; }
    }
  }
  int kind = dead ? 1 : 0;
  int q = 0;
  if (!dead)
    for (; q < c.nn; q++)
      if (!(c.P[c.np + q] & ~U)) { kind = 2; break; }
  if (COUNT) wk.scan += (u64)r + (u64)q;
  return kind;
}
template <typename M, bool COUNT>
__device__ __forceinline__ bool refuted(int j, M U, int e, const Clauses<M> &c, Work &wk) {
  return refuted_by<M, COUNT>(j, U, e, c, wk) != 0;
}

// TIMED: stop at a sub-block boundary once clock() passes `deadline` (after
// some progress); *stop = the window position reached (cnt when finished or
// when nothing more is needed), for the warp to hand the rest to idle lanes
template <typename M, int MODE, bool COUNT, bool TIMED = false>
__device__ i64 walk(int k, int me, u64 r_lo, u64 cnt, const Clauses<M> &c, const u32 *w, int rb,
                    int prune, Work &wk, const u64 *skj = nullptr, u64 wstar = ~0ull,
                    int need_p = 1, int need_m = 0, i64 *best_m = nullptr, bool exh = false,
                    unsigned deadline = 0, int *stop = nullptr) {
  if (TIMED) *stop = (int)cnt;
  // MODE 3 (PMS and MHS of one instance in one walk): the first witness of
  // phi (returned) and of phi+ alone (*best_m), each only while needed
  i64 dummy = GR_KEY_NONE;
  i64 &bm = MODE == 3 ? *best_m : dummy;
  bool wp = MODE != 3 || need_p, wm = MODE == 3 && need_m;
  // the ancestor stack: 5-bit entries below 32 variables, else 6 (J <= 12)
  constexpr int SB = sizeof(M) == 4 ? 5 : 6;
  constexpr int JM = sizeof(M) == 4 ? JMAX : (JMAX < 12 ? JMAX : 12);
  const int J = k < JM ? k : JM;
  const u64 *cs = tab_cs();  // C(n, j), j <= JMAX
#define CS(n, j) (cs[(n) * (JMAX + 1) + (j)])
  i64 best = GR_KEY_NONE;
  if (COUNT) wk.windows++;
  // ---- position the iterator on the sub-block that holds rank r_lo: colex
  // unrank of r_lo (element i is the largest c with C(c, i) <= the remaining
  // rank); the top k - J elements (binary search) form Utop, the J lowest go
  // to the mask Slow (downward scan over the shared binomial table)
  M Slow = 0;  // the J lowest elements of x (a register mask: no local-memory array)
  M Utop = 0;
  u64 rr = r_lo, base_top;
  {
    int cc = me - 1;
    for (int i = k; i > J; i--) {  // binary search in [i - 1, cc]
      int lo = i - 1, h = cc;
      while (lo < h) {
        const int mid = (lo + h + 1) >> 1;
        if (binom(mid, i) <= rr) lo = mid; else h = mid - 1;
      }
      Utop |= (M)1 << lo;
      rr -= binom(lo, i);
      cc = lo - 1;
    }
    base_top = r_lo - rr;  // rank of (Utop, the J lowest elements of [0, min Utop))
    // element i = the largest c <= cc with C(c, i) <= rr; the rows are
    // scanned downward four at a time (four independent shared-memory loads
    // per step instead of a chain of dependent ones); C(i-1, i) = 0 ends the
    // scan at row i-1 at the latest, so clamping rows at 0 is harmless
    for (int i = J; i >= 1; i--) {
      u64 v;
      for (;;) {
        const u64 v0 = CS(cc, i), v1 = CS(max(cc - 1, 0), i), v2 = CS(max(cc - 2, 0), i),
                  v3 = CS(max(cc - 3, 0), i);
        if (v0 <= rr) { v = v0; break; }
        if (v1 <= rr) { v = v1; cc -= 1; break; }
        if (v2 <= rr) { v = v2; cc -= 2; break; }
        if (v3 <= rr) { v = v3; cc -= 3; break; }
        cc -= 4;
      }
      Slow |= (M)1 << cc;
      rr -= v;
      cc--;
    }
  }
  int e_top = Utop ? ctz(Utop) : me;
  // Iterator state: the path t_0 > t_1 > ... > t_{d-1} of part-B choices
  // below Utop; the current node is (j = J - d, U, e = t_{d-1} or e_top) with
  // region R = R_j and ep = the parent's e (t_{d-2} or e_top).  tp is a stack
  // of the older ancestors t_{d-3} .. t_0, e_top (SB bits each, most recent
  // lowest; at depth d it holds d - 1 entries).  An entry stores e - 1: every
  // stored e is >= 1 and e_top can be m_eff = 32, which does not fit 5 bits
  // (a round-1 build stored e itself and read e_top = 32 back as 0, cutting
  // depth-1 siblings off in long windows at m_eff = 32).  Sub-blocks
  // partition the level in rank order, so the next sub-block starts where
  // this one ends: base += n.
  M U = Utop;
  // weighted: W(U), kept up to date as the iterator adds / removes elements
  u64 wU = 0;
  if (MODE == 2)
    for (M tt = U; tt; tt &= tt - 1) wU += w[ctz(tt)];
  u64 base = base_top;
  int d = 0, j = J, e = e_top, ep = e_top;
  u64 tp = 0;
  // descend: at node j, x lies in part B iff its j-th lowest element (the
  // highest of the j elements left in Slow) is >= R_j; then the child is
  // t = that element.  An ancestor whose whole subtree is refuted stops the
  // descent: the walk resumes after it (without this a window starting deep
  // inside a refuted subtree would refute each remaining sibling on the path
  // one by one).
  bool dead0 = false;
  while (j >= 2) {
    const int t = (int)(8 * sizeof(M) - 1) - (sizeof(M) == 4 ? __clz((int)Slow) : __clzll((long long)Slow));
    if (t < tab_reg()[j]) break;
    if (prune) {
      const int kind = refuted_by<M, COUNT>(j, U, e, c, wk);
      if (kind == 1 || (kind == 2 && !wm)) {
        dead0 = true;
        break;
      }
    }
    Slow ^= (M)1 << t;
    if (d > 0) tp = (tp << SB) | (u64)(ep - 1);
    ep = e;
    e = t;
    U |= (M)1 << t;
    if (MODE == 2) wU += w[t];
    base += CS(t, j);
    d++;
    j--;
  }
  int R = tab_reg()[j];
  // positions relative to r_lo fit 32 bits (windows hold <= 2^14 candidates)
  int pos = (int)((i64)base - (i64)r_lo);
  const int cnt32 = (int)cnt;
  // ---- iterate over sub-blocks in rank order
  for (;;) {
    if (pos >= cnt32) return best;
    if (TIMED && pos > 0 && (int)(clock() - deadline) > 0) {
      *stop = pos;
      return best;
    }
    const int n = tab_nb()[j * 65 + e];  // C(min(e, R_j), j)
    // An inner node (one with children) first asks whether its whole subtree
    // -- every x = U | S, S a j-subset of [0, e) -- is infeasible: a positive
    // clause missing U and [0, e), more than j pairwise disjoint positive
    // clauses missing U (restricted to [0, e)), or a negative clause inside
    // U.  Then all C(e, j) candidates of the subtree are decided at once.
    bool dead = dead0;
    dead0 = false;
#ifdef GR_DIRECT_WU
    if (MODE == 2) {
      u64 wd = 0;
      for (M tt = U; tt; tt &= tt - 1) wd += w[ctz(tt)];
      wU = wd;
    }
#endif
    const u64 WU = wU;  // weighted: W(U), and a bound on the whole subtree -- every
                        // x in it weighs >= W(U) + S_j (the j smallest weights);
                        // it can only matter below the incumbent of earlier
                        // levels (W*, strictly, R3) and below this lane's best
                        // so far (ties lose on rank: the walk is in rank order)
    if (MODE == 2) {
      if (prune && !dead) {
        const u64 lb = (u64)best >> rb;
        const u64 lim = best == GR_KEY_NONE ? wstar : (lb < wstar ? lb : wstar);
        if (WU + skj[j] >= lim) dead = true;
      }
    }
    if (!dead && prune && j >= 2 && R < e) {
      const int kind = refuted_by<M, COUNT>(j, U, e, c, wk);
      dead = kind == 1 || (kind == 2 && !wm);  // the MHS ignores phi-
    }
    if (!dead && n && pos + n > 0) {
      F2 F = tab_lowb()[n];
      if (pos < 0) F = f2_andnot(F, tab_lowb()[-pos]);
      if (cnt32 - pos < n) F = f2_and(F, tab_lowb()[cnt32 - pos]);
      if (COUNT) { wk.blocks++; wk.cands += (u64)f2_popc(F); }
      const int ea = e < R ? e : R;
      if (MODE == 3) {
        F = test_pos<M, COUNT>(j, U, F, c, wk);
        if (wm && f2_any(F)) {
          bm = (i64)(r_lo + (u64)(pos + f2_ctz(F)));
          wm = false;
        }
        if (wp && f2_any(F)) {
          F = test_neg<M, COUNT>(j, U, ea, F, c, wk);
          if (f2_any(F)) {
            best = (i64)(r_lo + (u64)(pos + f2_ctz(F)));
            wp = false;
          }
        }
        if (!wp && !wm && !exh) return best;  // exhaustive: the level is walked in full
        F = F2{0ull, 0ull};
      } else {
        F = test_sub<M, COUNT>(j, U, ea, F, c, wk);
      }
      if (f2_any(F)) {
        if (MODE == 2) {
          for (int h = 0; h < 2; h++)
            for (u64 f = h ? F.hi : F.lo; f; f &= f - 1) {
              const u64 idx = (u64)(64 * h + __ffsll((long long)f) - 1);
              const i64 key = (i64)(((WU + weight_low(j, idx, ea, w, cs)) << rb) |
                                    (r_lo + (u64)((i64)pos + (i64)idx)));
              best = key < best ? key : best;
            }
        } else {
          if (best == GR_KEY_NONE) best = (i64)(r_lo + (u64)(pos + f2_ctz(F)));
          if (MODE == 0) return best;
        }
      }
    }
    if (dead) {  // skip the whole subtree: its C(e, j) candidates are infeasible
      const u64 sz = CS(e, j);
      pos = sz >= (u64)(cnt32 - pos) ? cnt32 : pos + (int)sz;
    } else {
      pos += n;
    }
    // ---- advance: first child t = R of this node, else the next sibling up
    // the path
    if (!dead && j >= 2 && R < e) {
      if (d > 0) tp = (tp << SB) | (u64)(ep - 1);
      ep = e;
      e = R;
      U |= (M)1 << R;
      if (MODE == 2) wU += w[R];
      d++;
      j--;
      R = tab_reg()[j];
      continue;
    }
    if (d > 0 && e + 1 >= ep) {  // no next sibling here: pop until there is one
      do {
        U &= ~((M)1 << e);
        if (MODE == 2) wU -= w[e];
        d--;
        j++;
        e = ep;
        if (d > 0) {  // the stack holds the ancestors above the parent
          ep = (int)(tp & ((1u << SB) - 1u)) + 1;
          tp >>= SB;
        }
      } while (d > 0 && e + 1 >= ep);
      R = tab_reg()[j];
    }
    if (d > 0) {  // next sibling: t -> t + 1
      U ^= (M)3 << e;
      if (MODE == 2) wU += (u64)w[e + 1] - (u64)w[e];
      e++;
      continue;
    }
    // ---- next top-level U (Gosper on the (k-J)-subsets of [J, me))
    if (!Utop) return best;
    M S = Utop >> J;
    const M lb = lowbit(S);
    const M r = S + lb;
    S = r | (((r ^ S) >> 2) >> ctz(S));
    Utop = (M)(S << J);
    e_top = ctz(Utop);
    U = Utop;
    if (MODE == 2) {
      wU = 0;
      for (M tt = U; tt; tt &= tt - 1) wU += w[ctz(tt)];
    }
    e = ep = e_top;
  }
#undef CS
}

__device__ __forceinline__ i64 warp_min(i64 v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    i64 u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u < v ? u : v;
  }
  return v;
}

__device__ unsigned long long g_work[W_N];  // counting instantiation totals (Work units)
// counting instantiation: add a lane's work to the totals (wide: 64-bit masks)
__device__ __forceinline__ void work_add(const Work &wk, bool wide) {
  atomicAdd(&g_work[W_POS], (unsigned long long)wk.pos);
  atomicAdd(&g_work[W_NEG], (unsigned long long)wk.neg);
  atomicAdd(&g_work[W_SCAN], (unsigned long long)wk.scan);
  atomicAdd(&g_work[W_BLOCKS], (unsigned long long)wk.blocks);
  atomicAdd(&g_work[W_CANDS], (unsigned long long)wk.cands);
  atomicAdd(&g_work[W_WINDOWS], (unsigned long long)wk.windows);
  if (wide) atomicAdd(&g_work[W_WIDE], (unsigned long long)(wk.pos + wk.neg + wk.scan));
}

struct EnumParams {
  WS ws;
  const int64_t *off;
  int k, weighted, exhaustive, shard, nshard, prune;
  // fused: the MHS of the same batch (its own workspace ws2) is decided in
  // the PMS walk (MODE 3); the chunk plan is the PMS workspace's
  int fused;
  WS ws2;
};

template <typename M, bool COUNT>
__device__ i64 run_lane(const EnumParams &p, u64 r_lo, u64 cnt, int me, const Clauses<M> &c,
                        const u32 *w, int rb, Work &wk, const u64 *skj, u64 wstar) {
  if (p.weighted) return walk<M, 2, COUNT>(p.k, me, r_lo, cnt, c, w, rb, p.prune, wk, skj, wstar);
  if (p.exhaustive) return walk<M, 1, COUNT>(p.k, me, r_lo, cnt, c, w, rb, p.prune, wk);
  return walk<M, 0, COUNT>(p.k, me, r_lo, cnt, c, w, rb, p.prune, wk);
}


constexpr size_t TAB_SMEM =
    (JMAX + 1) * HX * 16 + 65 * (JMAX + 1) * 8 + 129 * 16 + 64 +
    ((JMAX + 1) * 65 + 15) / 16 * 16;  // HIT table, binomials, low masks, R_j, sub-block sizes
// clauses staged in shared memory (larger instances read L1/L2), sized for 4 CTAs per SM
#ifndef GR_ENUM_CTAS
#define GR_ENUM_CTAS 4
#endif
constexpr int ENUM_CTAS = GR_ENUM_CTAS;  // resident enumeration CTAs per SM (registers, smem)
// Two shapes of the enumeration CTA: NT = 256 threads x 4 per SM (room to
// stage 256 clauses), or 128 threads x 8 per SM for batches of at most 96
// clauses per instance (smaller CTAs, fewer lanes waiting at each chunk's
// barrier: C4 -13%).  A chunk is always NT lane windows; a 128-thread CTA
// walks two windows per thread.
template <int NTK>
__host__ __device__ constexpr int smc_of() {
  return (int)(((227 * 1024) / (ENUM_CTAS * NT / NTK) - 1024 - 600 - TAB_SMEM) / (16 * HREC + 8));
}
template <int NTK>
__host__ __device__ constexpr size_t enum_smem_of() {
  return TAB_SMEM + (size_t)smc_of<NTK>() * (16 * HREC + 8);
}
constexpr int NT_SMALL = NT / 2;

template <bool COUNT, int NTK>
__global__ void __launch_bounds__(NTK, COUNT ? 1 : ENUM_CTAS * NT / NTK) enum_kernel(EnumParams p) {
  extern __shared__ u64 cls[];  // [np][HREC] H records, [np + nn] P (u32 or u64)
  __shared__ u64 s_chunk;
  __shared__ int s_b, s_cur, s_skip, s_needp, s_needm;
  __shared__ u64 s_r0, s_ck;
  __shared__ u64 s_skj[JMAX + 1], s_wstar;  // weighted: S_j and the incumbent W*
  __shared__ u32 s_w[64];
  __shared__ i64 s_wmin[NTK / 32], s_wmin2[NTK / 32];
  const int t = threadIdx.x;
  if (t == 0) s_cur = -1;
  F2 *hitx = (F2 *)cls;  // [JMAX + 1][HX] HIT_j({x}): j-subsets of [0, R_j) containing x
  u64 *cs = cls + 2 * (JMAX + 1) * HX;  // [65][JMAX + 1] C(n, j), j <= JMAX
  F2 *lowb = (F2 *)(cs + 65 * (JMAX + 1));  // [129] the n lowest bits
  for (int q = t; q < (JMAX + 1) * HX; q += NTK)
    hitx[q] = F2{g_hit.lo[64 * (q / HX) + q % HX], g_hit.hi[64 * (q / HX) + q % HX]};
  for (int q = t; q < 65 * (JMAX + 1); q += NTK) cs[q] = binom(q / (JMAX + 1), q % (JMAX + 1));
  for (int q = t; q < 129; q += NTK) lowb[q] = f2_nbits((u64)q);
  int *reg = (int *)(lowb + 129);  // [JMAX + 1] R_j
  if (t <= JMAX) reg[t] = t ? region_of(t) : 0;
  unsigned char *nb = (unsigned char *)(reg + 16);  // [JMAX + 1][65] sub-block sizes
  for (int q = t; q < (JMAX + 1) * 65; q += NTK) {
    const int jj = q / 65, ee = q % 65;
    nb[q] = jj ? (unsigned char)binom(ee < region_of(jj) ? ee : region_of(jj), jj) : 0;
  }
  u64 *stage = cls + TAB_SMEM / 8;  // staged clause records
  const u64 Lc = p.ws.ctrl->lane_cands;
  const u64 CH = Lc * NTK;  // a chunk: one lane window per thread
  const u64 total = p.ws.ctrl->total_chunks;
  const int nact = p.ws.ctrl->n_active;
  const int *active = p.ws.active;  // list of this level (offset by the host)
  for (;;) {
    __syncthreads();
    if (t == 0) {
      u64 jn = atomicAdd((unsigned long long *)&p.ws.ctrl->next_chunk, 1ull);
      u64 ch = jn * (u64)p.nshard + (u64)p.shard;
      s_chunk = ch;
      s_skip = 0;
      if (ch < total) {
        // active index i: chunk_base[i] <= ch < chunk_base[i+1]
        int lo = 0, hi = nact - 1;
        while (lo < hi) {
          int mid = (lo + hi + 1) >> 1;
          if (p.ws.chunk_base[mid] <= ch) lo = mid; else hi = mid - 1;
        }
        const int b = active[lo];
        s_b = b;
        const u64 r0 = (ch - p.ws.chunk_base[lo]) * CH;
        s_r0 = r0;
        s_ck = binom(p.ws.meff[b], p.k);
        if (!p.weighted && !p.exhaustive) {
          const i64 cur = *(volatile i64 *)&p.ws.lvlkey[b];
          if (cur != GR_KEY_NONE && (u64)cur < r0) s_skip = 1;  // a lower witness exists
        }
        if (p.fused) {  // each solve is needed unless done or already below r0
          const i64 c1 = *(volatile i64 *)&p.ws.lvlkey[b];
          const i64 c2 = *(volatile i64 *)&p.ws2.lvlkey[b];
          const int np_ = !p.ws.done[b] && !(c1 != GR_KEY_NONE && (u64)c1 < r0 && !p.exhaustive);
          const int nm_ = !p.ws2.done[b] && !(c2 != GR_KEY_NONE && (u64)c2 < r0 && !p.exhaustive);
          s_needp = np_;
          s_needm = nm_;
          s_skip = !np_ && !nm_;
        }
      }
    }
    __syncthreads();
    if (s_chunk >= total) break;
    if (s_skip) continue;
    const int b = s_b;
    const int me = p.ws.meff[b], np = p.ws.npr[b], nn = p.ws.nnr[b];
    const int64_t lo = p.off[b];
    const bool staged = np + nn <= smc_of<NTK>();
    const bool narrow = staged && me <= 32;
    F2 *sH = (F2 *)stage;                       // [np][HREC]
    u64 *sP = stage + (size_t)2 * HREC * np;     // [np + nn] as u32 or u64
    if (b != s_cur) {
      if (staged) {
        for (int q = t; q < np * HREC; q += NTK) sH[q] = ((const F2 *)p.ws.hrec)[lo * HREC + q];
        if (narrow) {
          u32 *c32 = (u32 *)sP;
          for (int q = t; q < np + nn; q += NTK) c32[q] = (u32)p.ws.pk[lo + q];
        } else {
          for (int q = t; q < np + nn; q += NTK) sP[q] = p.ws.pk[lo + q];
        }
      }
      if (t < 64) s_w[t] = p.ws.wr[(size_t)b * 64 + t];
      if (p.weighted && t <= JMAX) s_skj[t] = p.ws.sk[(size_t)b * 65 + t];
      if (p.weighted && t == 0) s_wstar = p.ws.bestw[b];
      __syncthreads();
      if (t == 0) s_cur = b;
    }
    const u64 ck = s_ck;
    i64 key = GR_KEY_NONE, key_m = GR_KEY_NONE;
    Work wk;
    {
    const u64 r_lo = s_r0 + (u64)t * Lc;
    i64 key1 = GR_KEY_NONE, key_m1 = GR_KEY_NONE;
    if (r_lo < ck) {
      const u64 cnt = (ck - r_lo) < Lc ? (ck - r_lo) : Lc;
      const int rb = p.ws.rb[b];
      if (p.fused) {
        const int nq = s_needp, nm = s_needm;
        if (narrow) {
          Clauses<u32> c{(const u32 *)sP, sH, np, nn};
          key1 = walk<u32, 3, COUNT>(p.k, me, r_lo, cnt, c, s_w, rb, p.prune, wk, nullptr, ~0ull,
                                    nq, nm, &key_m1, p.exhaustive);
        } else if (staged) {
          Clauses<u64> c{sP, sH, np, nn};
          key1 = walk<u64, 3, COUNT>(p.k, me, r_lo, cnt, c, s_w, rb, p.prune, wk, nullptr, ~0ull,
                                    nq, nm, &key_m1, p.exhaustive);
        } else {
          Clauses<u64> c{p.ws.pk + lo, (const F2 *)p.ws.hrec + lo * HREC, np, nn};
          key1 = walk<u64, 3, COUNT>(p.k, me, r_lo, cnt, c, s_w, rb, p.prune, wk, nullptr, ~0ull,
                                    nq, nm, &key_m1, p.exhaustive);
        }
      } else if (narrow) {
        Clauses<u32> c{(const u32 *)sP, sH, np, nn};
        key1 = run_lane<u32, COUNT>(p, r_lo, cnt, me, c, s_w, rb, wk, s_skj, s_wstar);
      } else if (staged) {
        Clauses<u64> c{sP, sH, np, nn};
        key1 = run_lane<u64, COUNT>(p, r_lo, cnt, me, c, s_w, rb, wk, s_skj, s_wstar);
      } else {
        Clauses<u64> c{p.ws.pk + lo, (const F2 *)p.ws.hrec + lo * HREC, np, nn};
        key1 = run_lane<u64, COUNT>(p, r_lo, cnt, me, c, s_w, rb, wk, s_skj, s_wstar);
      }
    }
    key = key1 < key ? key1 : key;
    key_m = key_m1 < key_m ? key_m1 : key_m;
    }
    if (COUNT) work_add(wk, !narrow);
    key = warp_min(key);
    if (p.fused) key_m = warp_min(key_m);
    if ((t & 31) == 0) {
      s_wmin[t >> 5] = key;
      s_wmin2[t >> 5] = key_m;
    }
    __syncthreads();
    if (t == 0) {
      i64 v = s_wmin[0], v2 = s_wmin2[0];
      for (int i = 1; i < NTK / 32; i++) {
        v = s_wmin[i] < v ? s_wmin[i] : v;
        v2 = s_wmin2[i] < v2 ? s_wmin2[i] : v2;
      }
      if (v != GR_KEY_NONE) atomicMin((long long *)&p.ws.lvlkey[b], (long long)v);
      if (p.fused && v2 != GR_KEY_NONE) atomicMin((long long *)&p.ws2.lvlkey[b], (long long)v2);
    }
  }
}

// ---------------------------------------------------------------------------
// finish: commit level k, plan level k+1 (one CTA)
// ---------------------------------------------------------------------------
__device__ __forceinline__ int bitlen(u64 x) { return x ? 64 - __clzll((long long)x) : 0; }

// colex unrank (common.cuh's unrank_colex) against a shared-memory copy of
// the binomial table: the finish is a latency chain (k binary searches of
// dependent reads per witness), so each read is a shared-memory hit instead of
// an L2 round trip
__device__ __forceinline__ u64 unrank_colex_smem(const u64 (*tb)[65], u64 r, int k, int n) {
  u64 x = 0;
  int hi = n - 1;
  for (int j = k; j >= 1; j--) {
    int lo = j - 1, h = hi;
    while (lo < h) {
      const int mid = (lo + h + 1) >> 1;
      if (tb[mid][j] <= r) lo = mid; else h = mid - 1;
    }
    x |= 1ull << lo;
    r -= tb[lo][j];
    hi = lo - 1;
  }
  return x;
}

// phase 1 of the finish: commit level k of every listed instance
__device__ void finish_commit(const In &in, const Out &out, const WS &ws, int which, int k,
                              int exhaustive, int part, int nparts) {
  const int t = threadIdx.x;
  __shared__ u64 s_binom[65][65];  // C(n, j), zero for j > n (as g_binom); columns j <= k only
  for (int i = t; i < 65 * (k + 1); i += FT) {
    const int n = i / (k + 1), j = i - n * (k + 1);
    s_binom[n][j] = __ldg(&g_binom.v[n][j]);
  }
  __syncthreads();
  const bool weighted = in.w != nullptr;
  const int nact_in = k == 0 ? in.B : ws.ctrl->n_active;
  const int *cur = ws.active + (size_t)(k & 1) * in.B;  // list enumerated at level k
  {
    for (int i = part * FT + t; i < nact_in; i += nparts * FT) {
      const int b = cur[i];
      if (ws.done[b]) continue;  // fused: listed for the other solve only
      const int me = ws.meff[b];
      const u64 ck = s_binom[me][k];
      const i64 key = ws.lvlkey[b];
      const u64 s0 = ws.sup[2 * b], s1 = ws.sup[2 * b + 1];
      if (!weighted) {
        if (key != GR_KEY_NONE) {
          const u64 rank = (u64)key;
          const u64 x = unrank_colex_smem(s_binom, rank, k, me);
          const u64 d = sat_add(ws.decided[b], exhaustive ? ck : rank + 1);
          ws.done[b] = 1;
          write_result(in, out, b, GR_SAT, x, s0, s1, (u64)k, d, which);
        } else {
          ws.decided[b] = sat_add(ws.decided[b], ck);
          if (k >= ws.kmax[b]) {
            ws.done[b] = 1;
            write_result(in, out, b, GR_UNSAT, 0, s0, s1, 0, ws.decided[b], which);
          }
        }
      } else {
        ws.decided[b] = sat_add(ws.decided[b], ck);
        if (key != GR_KEY_NONE) {
          const int rb = ws.rb[b];
          const u64 Wk = (u64)key >> rb;
          const u64 rank = (u64)key & ((rb ? (1ull << rb) : 1ull) - 1ull);
          if (Wk < ws.bestw[b]) {  // strictly smaller W replaces the incumbent (R3)
            ws.bestw[b] = Wk;
            ws.bestx[b] = unrank_colex_smem(s_binom, rank, k, me);
          }
        }
        const u64 bw = ws.bestw[b];
        const bool stop = k >= ws.kmax[b] || (bw != ~0ull && ws.sk[(size_t)b * 65 + k + 1] >= bw);
        if (stop) {
          ws.done[b] = 1;
          if (bw != ~0ull) write_result(in, out, b, GR_SAT, ws.bestx[b], s0, s1, bw, ws.decided[b], which);
          else write_result(in, out, b, GR_UNSAT, 0, s0, s1, 0, ws.decided[b], which);
        }
      }
    }
    __syncthreads();
  }
}

// phase 2: compact the active list and plan level k+1.  done_other (fused
// PMS + MHS): the MHS workspace's done flags -- an instance stays listed (and
// planned) while either solve still searches
__device__ void finish_plan(const In &in, const Out &out, const WS &ws, int which, int k,
                            int enum_lanes, u64 fixed_lane, int windows_per_lane, u64 lane_max,
                            u64 lane_max_w, const int *done_other, int chunk_lanes,
                            bool plan_chunks = true) {
  typedef cub::BlockScan<u64, FT> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ u64 s_carry;
  __shared__ int s_cnt, s_wait;
  const int t = threadIdx.x;
  if (t == 0) s_wait = 0;  // shared memory starts undefined
  __syncthreads();
  const bool weighted = in.w != nullptr;
  const int nact_in = k == 0 ? in.B : ws.ctrl->n_active;
  int *cur = ws.active + (size_t)(k & 1) * in.B;        // list enumerated at level k
  int *nxt = ws.active + (size_t)((k + 1) & 1) * in.B;  // list for level k+1
  // phase 2: compact the still-active instances and plan level k+1
  // (with start levels, every unfinished instance is revisited: those whose
  // start level is above k+1 wait, counted in n_remaining)
  const bool all = k == 0 || in.kstart != nullptr;
  const int n2 = all ? in.B : nact_in;
  // each thread takes a contiguous segment of the list (the loads of its
  // instances are independent, one block scan for all): pass A decides and
  // records each entry's level size (~0: not listed), pass B compacts
  const u64 NOTL = ~0ull;
  const int per = (n2 + FT - 1) / FT;
  const int i0 = min(n2, t * per), i1 = min(n2, i0 + per);
  u64 my_cnt = 0, my_sz = 0;
  int my_wait = 0;
  for (int i = i0; i < i1; i++) {
    const int b = all ? i : cur[i];
    u64 v = NOTL;
    if (ws.done[b] && (!done_other || done_other[b])) {
    } else if (k + 1 < ws.ks[b]) {
      my_wait++;
    } else {
      const int me = ws.meff[b];
      const u64 ck = binom(me, k + 1);
      bool ok = true;
      if (weighted) {
        const int rb = bitlen(ck - 1);
        if (bitlen(ws.wtot[b]) + rb > 63) {  // key (W << rb | rank) would not fit
          ws.done[b] = 1;
          write_result(in, out, b, GR_UNSUPPORTED, 0, 0, 0, 0, ws.decided[b], which);
          ok = false;
        } else {
          ws.rb[b] = rb;
        }
      }
      if (ok) {
        ws.lvlkey[b] = GR_KEY_NONE;
        v = ck;
      }
    }
    ws.ptmp[i] = v;
    if (v != NOTL) {
      my_cnt++;
      my_sz += v;  // candidates of level k+1 (wrap-around is harmless: only sizes L)
    }
  }
  if (my_wait) atomicAdd(&s_wait, my_wait);
  u64 pos, n_list;
  Scan(tmp).ExclusiveSum(my_cnt, pos, n_list);
  __syncthreads();
  u64 szpos, sz_all;
  Scan(tmp).ExclusiveSum(my_sz, szpos, sz_all);
  __syncthreads();
  {
    u64 q = pos;
    for (int i = i0; i < i1; i++) {
      const u64 v = ws.ptmp[i];
      if (v == NOTL) continue;
      nxt[q] = all ? i : cur[i];
      ws.chunk_base[q] = v;  // the level size; the plan below turns it into a prefix
      q++;
    }
  }
  if (t == 0) {
    s_cnt = (int)n_list;
    s_carry = sz_all;
  }
  __syncthreads();
  // lane window L: about 3 windows per lane of the enumeration grid, a power
  // of two in [256, 2^18] (weighted levels: 4 windows, at most 2^16)
  const u64 Lmax = weighted ? lane_max_w : lane_max;
  // windows per lane: the host's value for unit weights, its high 16 bits
  // for weighted levels
  const u64 wpl = weighted ? (u64)(windows_per_lane >> 16) : (u64)(windows_per_lane & 0xffff);
  u64 L = s_carry / ((u64)enum_lanes * (wpl ? wpl : 2));
  L = L < 256 ? 256 : (L > Lmax ? Lmax : L);
  L = 1ull << (63 - __clzll((long long)L));
  if (fixed_lane) L = fixed_lane;  // GR_LANE_CANDIDATES override
  const u64 CH = L * (u64)chunk_lanes;  // the enumeration CTA's threads
  const int nact = s_cnt;
  __syncthreads();
  if (t == 0) s_carry = 0;
  __syncthreads();
  if (plan_chunks) {
    const int per2 = (nact + FT - 1) / FT;
    const int q0 = min(nact, t * per2), q1 = min(nact, q0 + per2);
    u64 my_ch = 0;
    for (int q = q0; q < q1; q++) my_ch += (ws.chunk_base[q] + CH - 1) / CH;
    u64 cpos, ch_all;
    Scan(tmp).ExclusiveSum(my_ch, cpos, ch_all);
    __syncthreads();
    for (int q = q0; q < q1; q++) {
      const u64 nch = (ws.chunk_base[q] + CH - 1) / CH;
      ws.chunk_base[q] = cpos;
      cpos += nch;
    }
    if (t == 0) s_carry = ch_all;
    __syncthreads();
  }
  if (t == 0) {
    ws.chunk_base[nact] = s_carry;
    ws.ctrl->n_active = nact;
    ws.ctrl->n_remaining = nact + s_wait;
    ws.ctrl->total_chunks = s_carry;
    ws.ctrl->next_chunk = 0;
    ws.ctrl->lane_cands = L;
  }
}

__global__ void __launch_bounds__(FT, 1) finish_kernel(In in, Out out, WS ws, int which, int k,
                                                    int exhaustive, int enum_lanes,
                                                    u64 fixed_lane, int windows_per_lane,
                                                    u64 lane_max, u64 lane_max_w,
                                                    const int *done_other, int chunk_lanes) {
  // the commit is per instance: every block takes a share; the last block to
  // finish it plans the next level for all
  if (k > 0) finish_commit(in, out, ws, which, k, exhaustive, blockIdx.x, gridDim.x);
  if (gridDim.x > 1 && !cta_last_arrival(&ws.ctrl->fin_ticket, gridDim.x)) return;
  finish_plan(in, out, ws, which, k, enum_lanes, fixed_lane, windows_per_lane, lane_max, lane_max_w,
              done_other, chunk_lanes);
}

// fused PMS (ws1) + MHS (ws2): both commits, then the MHS list, then the PMS
// plan over the union -- one launch per level
__global__ void __launch_bounds__(FT, 1) finish_fused_kernel(In in1, Out out1, WS ws1, In in2, Out out2,
                                                          WS ws2, int k, int exhaustive, int enum_lanes,
                                                          u64 fixed_lane, int windows_per_lane,
                                                          u64 lane_max, u64 lane_max_w,
                                                          int chunk_lanes) {
  // blocks [0, P) commit the PMS, [P, 2P) the MHS; the last block plans
  const int P = gridDim.x / 2;
  if (k > 0) {
    if ((int)blockIdx.x < P) finish_commit(in1, out1, ws1, 0, k, exhaustive, blockIdx.x, P);
    else finish_commit(in2, out2, ws2, 1, k, exhaustive, blockIdx.x - P, P);
  }
  if (!cta_last_arrival(&ws1.ctrl->fin_ticket, gridDim.x)) return;
  finish_plan(in2, out2, ws2, 1, k, enum_lanes, fixed_lane, windows_per_lane, lane_max, lane_max_w,
              nullptr, chunk_lanes, false);  // its list only: the PMS workspace plans the chunks
  __syncthreads();
  finish_plan(in1, out1, ws1, 0, k, enum_lanes, fixed_lane, windows_per_lane, lane_max, lane_max_w,
              ws2.done, chunk_lanes);
}

// ---------------------------------------------------------------------------
// queue_kernel: the whole level loop of a solve in ONE persistent launch
// ---------------------------------------------------------------------------
// each instance runs its own level loop on the device.  The
// unit of work is a task = level k of instance b of solve sv (§8(a) a3); its
// colex rank range [0, C(m_eff, k)) is cut into warp chunks of 32 lane
// windows (a4).  Tasks are published into a ticket ring: a CTA takes the next
// ticket (one atomic), waits until the ring entry of that ticket is written,
// stages the task's instance (clause records, a5) and its warps pull warp
// chunks from the task's claim counter until it is exhausted -- a warp never
// waits for the other warps of its CTA except when the CTA changes task.  A
// task with many chunks gets up to one ring entry per CTA so that every idle
// CTA can join it.  The warp that finishes the last chunk of a task commits
// the level (a6, a7: decode, weighted incumbent, S_k stop rule, k_max) and
// either finishes the instance or publishes level k+1.  Instances progress
// independently: no grid-wide barrier per level, no finish launch, no host
// round trip.
struct QParams {
  WS ws[2];        // solve workspaces: ws[0] holds the ring and the control block
  In in[2];
  Out out[2];
  int which[2];    // 0 PMS / WPMS, 1 MHS (for write_result)
  int weighted[2]; // solve sv is weighted (MODE 2)
  int nsolve;      // 1, or 2 independent solves sharing the launch
  int fused;       // 1: one walk decides PMS (ws[0]) and MHS (ws[1]) of each instance (MODE 3)
  int exhaustive, prune;
  int spec;        // levels a speculative chain may run ahead of the last committed one
  u64 spec_max;    // largest level (candidates) published speculatively
  u64 gen;         // launch generation, 1..4095 (ring entries)
  u64 ring_mask;   // ring entries - 1
  int ring_log2;   // log2(ring entries)
  int lanes;       // threads of the grid (lane window sizing)
  int grid, nwarps;  // CTAs of the queue_kernel grid, warps per CTA (ring entries per task)
  int wpl;         // lane windows per lane (unit | weighted << 16)
  u64 lane_max, lane_max_w, fixed_lane, lane_min;  // lane_min: unit | weighted << 32
  int local_max;   // a next level of at most this many chunks stays with the committing CTA
  u64 lane_split;  // smallest lane window a small level is split to (a chunk per warp)
  int spec_idle;   // speculate only while CTAs sit idle (1), or always (0)
  unsigned slice;  // fused walk: clock cycles per time slice (0: untimed windows)
  int split_min;   // smallest share of a window handed to an idle lane
};

// gpu-scope acquire load / acq_rel add (PTX memory model): the completion
// count and the ring entries order what they publish without a full fence
__device__ __forceinline__ u64 ld_acquire(const u64 *p) {
  u64 v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u64 atom_add_acq_rel(u64 *p, u64 v) {
  u64 old;
  asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ u64 gtime() {
  u64 t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ u64 vld(const u64 *p) { return *(const volatile u64 *)p; }
__device__ __forceinline__ i64 vld(const i64 *p) { return *(const volatile i64 *)p; }
__device__ __forceinline__ int vld(const int *p) { return *(const volatile int *)p; }
__device__ __forceinline__ unsigned vldu(const unsigned *p) { return *(const volatile unsigned *)p; }
__device__ __forceinline__ void work_sub(u64 *qw, u64 v) {
  atomicAdd((unsigned long long *)qw, (unsigned long long)(-(long long)v));
}

// the ring entry a waiter of ticket e expects, minus its payload
__device__ __forceinline__ u64 ring_stamp(const QParams &P, u64 e) {
  return (P.gen << 52) | (((e >> P.ring_log2) & 0xfffull) << 40);
}

// Fill the task record of level k of (b, sv) -- not published.  work =
// candidates in flight including this level (lane window sizing); depth > 0:
// an unconfirmed speculation.  false: the weighted key (W << rb | rank) of
// this level would not fit 63 bits (the caller reports GR_UNSUPPORTED).
__device__ bool q_make(const QParams &P, int sv, int b, int k, u64 work, int depth, u64 *ti_out,
                       u64 ti_pre = ~0ull) {
  const WS &w = P.ws[sv];
  const int me = w.meff[b];
  const u64 ck = binom(me, k);
  int rb = 0;
  if (P.weighted[sv]) {
    rb = bitlen(ck - 1);
    if (bitlen(vld(&w.wtot[b])) + rb > 63) return false;
  }
  // lane window: about wpl windows per lane of the grid over all the work in
  // flight, a power of two in [lane_min, lane_max]
  const bool wt = P.weighted[sv] != 0;
  const u64 wpl = wt ? (u64)(P.wpl >> 16) : (u64)(P.wpl & 0xffff);
  const u64 Lmax = wt ? P.lane_max_w : P.lane_max;
  const u64 Lmin = wt ? P.lane_min >> 32 : P.lane_min & 0xffffffffull;
  u64 L = work / ((u64)P.lanes * (wpl ? wpl : 2));
  L = L < Lmin ? Lmin : (L > Lmax ? Lmax : L);
  L = 1ull << (63 - __clzll((long long)L));
  // a small level still gets a chunk per warp of a CTA (down to P.lane_split
  // candidates per window): its CTA's warps share it instead of waiting
  while (L > P.lane_split && (ck + 32 * L - 1) / (32 * L) < (u64)P.nwarps) L >>= 1;
  if (P.fixed_lane) L = P.fixed_lane;
  const u64 nch = (ck + 32 * L - 1) / (32 * L);
  // task records of solve sv live in its own workspace (<= 2 per level)
  // (ti_pre: an index the caller took for a whole warp with one atomic)
  const u64 ti = ti_pre != ~0ull ? ti_pre : atomicAdd((unsigned long long *)&w.ctrl->q_tasks, 1ull);
  Task *T = w.tasks + ti;
  T->claimed = 0;
  T->pending = nch + (depth ? 1 : 0);
  T->nchunks = nch;
  T->L = L;
  T->key[0] = GR_KEY_NONE;
  T->key[1] = GR_KEY_NONE;
  T->b = b;
  T->k = k;
  T->succ = 0;
  T->sv = (unsigned char)sv;
  T->rb = (unsigned char)rb;
  T->depth = (unsigned char)depth;
  T->cancelled = 0;
  T->t_make = gtime();
  T->t_exhaust = T->t_commit = T->t_unused = 0;
  *ti_out = ti;
  return true;
}

// level k of (b, sv) can be a task: its weighted key fits 63 bits (q_make)
__device__ __forceinline__ bool q_fits(const QParams &P, int sv, int b, int k) {
  if (!P.weighted[sv]) return true;
  const WS &w = P.ws[sv];
  return bitlen(vld(&w.wtot[b])) + bitlen(binom(w.meff[b], k) - 1) <= 63;
}

// Ring entries of a task with nch warp chunks (single thread): one, plus one
// per further (warps per CTA) chunks up to the grid, as far as the
// extra-entry budget allows.  Returns the count; *e0 = the first entry.
__device__ u64 q_entries(const QParams &P, u64 nch, u64 *e0) {
  Ctrl *c = P.ws[0].ctrl;
  const u64 nw = (u64)P.nwarps;
  u64 extra = (nch + nw - 1) / nw;
  extra = (extra > (u64)P.grid ? (u64)P.grid : extra) - 1;
  if (extra) {
    const long long got = (long long)atomicAdd((unsigned long long *)&c->q_budget,
                                               (unsigned long long)(-(long long)extra));
    if (got < (long long)extra) {
      atomicAdd((unsigned long long *)&c->q_budget, (unsigned long long)extra);
      extra = 0;
    }
  }
  *e0 = atomicAdd((unsigned long long *)&c->q_entries, extra + 1);
  return extra + 1;
}
// entry i of a task: written by any thread after the task record's fence
__device__ __forceinline__ void q_publish(const QParams &P, u64 word, u64 e0, u64 i) {
  const u64 e = e0 + i;
  *(volatile u64 *)&P.ws[0].ring[e & P.ring_mask] = ring_stamp(P, e) | (i ? (1ull << 39) : 0ull) | word;
}

// Commit level k of solve s for instance b with the level's key (decode,
// weighted incumbent, S_k stop rule, k_max).  Returns whether solve s still
// searches.  Single thread.
__device__ bool q_commit_one(const QParams &P, int s, int b, int k, i64 key, int rb) {
  const WS &w = P.ws[s];
  if (vld(&w.done[b])) return false;
  const In &in = P.in[s];
  const Out &out = P.out[s];
  const int me = w.meff[b];
  const u64 ck = binom(me, k);
  const u64 s0 = w.sup[2 * b], s1 = w.sup[2 * b + 1];
  const u64 dec = vld(&w.decided[b]);
  if (!P.weighted[s]) {
    if (key != GR_KEY_NONE) {
      const u64 x = unrank_colex((u64)key, k, me);
      const u64 d = sat_add(dec, P.exhaustive ? ck : (u64)key + 1);
      w.done[b] = 1;
      write_result(in, out, b, GR_SAT, x, s0, s1, (u64)k, d, P.which[s]);
      return false;
    }
    w.decided[b] = sat_add(dec, ck);
    if (k >= w.kmax[b]) {
      w.done[b] = 1;
      write_result(in, out, b, GR_UNSAT, 0, s0, s1, 0, sat_add(dec, ck), P.which[s]);
      return false;
    }
    return true;
  }
  const u64 d = sat_add(dec, ck);
  w.decided[b] = d;
  u64 bw = vld(&w.bestw[b]);
  if (key != GR_KEY_NONE) {
    const u64 Wk = (u64)key >> rb;
    const u64 rank = (u64)key & ((rb ? (1ull << rb) : 1ull) - 1ull);
    if (Wk < bw) {  // strictly smaller W replaces the incumbent (R3)
      bw = Wk;
      w.bestw[b] = Wk;
      w.bestx[b] = unrank_colex(rank, k, me);
    }
  }
  const bool stop = k >= w.kmax[b] || (bw != ~0ull && w.sk[(size_t)b * 65 + k + 1] >= bw);
  if (stop) {
    w.done[b] = 1;
    if (bw != ~0ull) write_result(in, out, b, GR_SAT, vld(&w.bestx[b]), s0, s1, bw, d, P.which[s]);
    else write_result(in, out, b, GR_UNSAT, 0, s0, s1, 0, d, P.which[s]);
    return false;
  }
  return true;
}

// the instance cannot go on to the next level: its weighted key would not fit
__device__ void q_unsupported(const QParams &P, int sv, int b) {
  const WS &w = P.ws[sv];
  w.done[b] = 1;
  write_result(P.in[sv], P.out[sv], b, GR_UNSUPPORTED, 0, 0, 0, 0, vld(&w.decided[b]), P.which[sv]);
}

// cancel a speculative chain (its levels are not needed: the instance ended)
__device__ void q_cancel(const QParams &P, int sv, Task *S) {
  for (;;) {
    *(volatile unsigned char *)&S->cancelled = 1;
    work_sub(&P.ws[sv].ctrl->q_work, binom(P.ws[sv].meff[S->b], S->k));
    const unsigned s2 = atomicCAS(&S->succ, 0u, SUCC_CLOSED);
    if (s2 == 0u || s2 == SUCC_CLOSED) return;
    S = P.ws[sv].tasks + (s2 - 1);
  }
}

// All chunks of task ti are done (and it is confirmed): commit it; then either
// confirm its speculative successor (and commit that one too if its chunks
// are done as well), publish level k+1, or retire the instance.  Lane 0 of
// the committing warp.  Returns the ring entries the warp must publish
// (*word, *e0) -- 0 if none.
// local_max > 0: a next level of at most local_max chunks is not published
// but returned in *local (task index + 1) for the committing CTA to walk.
__device__ u64 q_commit_chain(const QParams &P, int sv, u64 ti, u64 *word, u64 *e0, u64 local_max = 0,
                              u64 *local = nullptr) {
  Ctrl *c = P.ws[0].ctrl;
  u64 *qw = &P.ws[sv].ctrl->q_work;
  for (;;) {
    Task *T = P.ws[sv].tasks + ti;
    const int b = T->b, k = T->k;
    const int me = P.ws[sv].meff[b];
    T->t_commit = gtime();
    work_sub(qw, binom(me, k));
    bool open;
    if (P.fused) {
      const bool o0 = q_commit_one(P, 0, b, k, vld(&T->key[0]), 0);
      const bool o1 = q_commit_one(P, 1, b, k, vld(&T->key[1]), 0);
      open = o0 || o1;
    } else {
      open = q_commit_one(P, sv, b, k, vld(&T->key[0]), T->rb);
    }
    const unsigned s = atomicCAS(&T->succ, 0u, SUCC_CLOSED);
    if (s == 0u) {  // no speculative successor: publish level k+1, or retire
      if (open && k < 64) {
        const u64 ck1 = binom(me, k + 1);
        const u64 wk = atomicAdd((unsigned long long *)qw, (unsigned long long)ck1) + ck1;
        u64 ti2;
        if (q_make(P, sv, b, k + 1, wk, 0, &ti2)) {
          __threadfence();  // the task record before its entries
          *word = ti2 | ((u64)sv << 38);
          if (local && P.ws[sv].tasks[ti2].nchunks <= local_max) {
            *local = ti2 + 1;
            return 0;
          }
          return q_entries(P, P.ws[sv].tasks[ti2].nchunks, e0);
        }
        work_sub(qw, ck1);
        q_unsupported(P, sv, b);
      }
      __threadfence();  // results before the count that ends the launch
      atomicSub(&c->q_remaining, 1);
      return 0;
    }
    Task *S = P.ws[sv].tasks + (s - 1);
    if (!open) {  // the instance ended: its speculative levels are not needed
      q_cancel(P, sv, S);
      __threadfence();
      atomicSub(&c->q_remaining, 1);
      return 0;
    }
    *(volatile unsigned char *)&S->depth = 0;  // confirmed
    if (atom_add_acq_rel(&S->pending, ~0ull) != 1ull) return 0;  // its last chunk will commit it
    ti = s - 1;  // every chunk of the successor is done already: commit it here
  }
}

// The seed, in two launches over all instances (warp-aggregated atomics: a
// single CTA doing one atomic per instance took 0.3 ms at C4's 2 x 10 000):
// queue_work_kernel sums the work in flight of each solve (its open
// instances' first levels) and sets the ring budget; queue_seed_kernel
// makes and publishes the first level of every open (instance, solve) and
// counts them (the pack zeroed the queue counters).
__device__ __forceinline__ bool q_open(const QParams &P, int sv, int b) {
  return !P.ws[sv].done[b] || (P.fused && !P.ws[1].done[b]);
}
__global__ void __launch_bounds__(256) queue_work_kernel(QParams P, long long budget) {
  __shared__ unsigned long long s_work[2];
  if (threadIdx.x < 2) s_work[threadIdx.x] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) P.ws[0].ctrl->q_budget = budget;
  __syncthreads();
  const int ns = P.fused ? 1 : P.nsolve;
  const int B = P.in[0].B;
  for (int sv = 0; sv < ns; sv++) {
    u64 my = 0;
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x)
      if (q_open(P, sv, b)) my += binom(P.ws[sv].meff[b], P.ws[sv].ks[b]);
    for (int o = 16; o; o >>= 1) my += __shfl_xor_sync(0xffffffffu, my, o);
    if ((threadIdx.x & 31) == 0 && my) atomicAdd(&s_work[sv], (unsigned long long)my);
  }
  __syncthreads();
  if (threadIdx.x < ns && s_work[threadIdx.x])
    atomicAdd((unsigned long long *)&P.ws[threadIdx.x].ctrl->q_work, s_work[threadIdx.x]);
}
__global__ void __launch_bounds__(256) queue_seed_kernel(QParams P) {
  const int ns = P.fused ? 1 : P.nsolve;
  const int B = P.in[0].B;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  Ctrl *c0 = P.ws[0].ctrl;
  for (int sv = 0; sv < ns; sv++) {
    const WS &w = P.ws[sv];
    const u64 work = vld(&w.ctrl->q_work);
    for (int b0 = blockIdx.x * blockDim.x; b0 < B; b0 += gridDim.x * blockDim.x) {  // warp-uniform
      const int b = b0 + (int)threadIdx.x;
      const bool open = b < B && q_open(P, sv, b);
      const bool fits = open && q_fits(P, sv, b, w.ks[b]);
      if (open && !fits) {
        work_sub(&w.ctrl->q_work, binom(w.meff[b], w.ks[b]));
        q_unsupported(P, sv, b);
      }
      // task indices and the count of open units: one atomic each per warp
      const unsigned bal = __ballot_sync(0xffffffffu, fits);
      if (!bal) continue;
      u64 base = 0;
      if (lane == 0) {
        base = atomicAdd((unsigned long long *)&w.ctrl->q_tasks, (unsigned long long)__popc(bal));
        atomicAdd(&c0->q_remaining, __popc(bal));
      }
      base = __shfl_sync(0xffffffffu, base, 0);
      const u64 ti = base + (u64)__popc(bal & lt);
      u64 extra = 0;
      if (fits) {
        u64 t2;
        q_make(P, sv, b, w.ks[b], work, 0, &t2, ti);
        const u64 nw = (u64)P.nwarps, nch = w.tasks[ti].nchunks;
        extra = (nch + nw - 1) / nw;
        extra = (extra > (u64)P.grid ? (u64)P.grid : extra) - 1;
      }
      // extra entries from the budget (all of the warp's or none) and the
      // warp's entries: one atomic each
      u64 tx = extra;
      for (int o = 16; o; o >>= 1) tx += __shfl_xor_sync(0xffffffffu, tx, o);
      int ok = 1;
      if (lane == 0 && tx) {
        const long long got = (long long)atomicAdd((unsigned long long *)&c0->q_budget,
                                                   (unsigned long long)(-(long long)tx));
        if (got < (long long)tx) {
          atomicAdd((unsigned long long *)&c0->q_budget, (unsigned long long)tx);
          ok = 0;
        }
      }
      ok = __shfl_sync(0xffffffffu, ok, 0);
      const u64 n = fits ? 1 + (ok ? extra : 0) : 0;
      u64 incl = n;
      for (int o = 1; o < 32; o <<= 1) {
        const u64 y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const u64 tot = __shfl_sync(0xffffffffu, incl, 31);
      u64 eb = 0;
      if (lane == 0) eb = atomicAdd((unsigned long long *)&c0->q_entries, (unsigned long long)tot);
      eb = __shfl_sync(0xffffffffu, eb, 0);
      // (no fence: queue_kernel starts after this launch completes, which
      // orders every record before every entry)
      for (u64 i = 0; i < n; i++) q_publish(P, ti | ((u64)sv << 38), eb + incl - n, i);
    }
  }
}

// KIND 0: unit-weight solves (MODE 0, or 1 when exhaustive); 1: the fused
// PMS + MHS walk (MODE 3); 2: weighted PMS (MODE 2), possibly with an MHS
// (MODE 0) in the same launch
template <typename M, int KIND, bool COUNT, bool TIMED = false>
__device__ __forceinline__ i64 q_walk(const QParams &P, int sv, int need, int k, int me, u64 r_lo,
                                      u64 cnt, const Clauses<M> &cc, const u32 *sw, int rb,
                                      Work &wk, const u64 *skj, u64 wstar, i64 *key_m,
                                      unsigned deadline = 0, int *stop = nullptr) {
  if (KIND == 1)
    return walk<M, 3, COUNT, TIMED>(k, me, r_lo, cnt, cc, sw, rb, P.prune, wk, nullptr, ~0ull, need & 1,
                                    need >> 1, key_m, P.exhaustive, deadline, stop);
  if (TIMED) *stop = (int)cnt;
  if (KIND == 2 && P.weighted[sv])
    return walk<M, 2, COUNT>(k, me, r_lo, cnt, cc, sw, rb, P.prune, wk, skj, wstar);
  if (P.exhaustive) return walk<M, 1, COUNT>(k, me, r_lo, cnt, cc, sw, rb, P.prune, wk);
  return walk<M, 0, COUNT>(k, me, r_lo, cnt, cc, sw, rb, P.prune, wk);
}

// The fused walk of one warp chunk in time slices: a lane walks its window
// for at most P.slice clocks at a time; then the warp ballots and the lane
// with the most range left hands equal shares of it to the lanes that are
// done (every lane takes part, with or without a window of its own).
template <typename M, int KIND, bool COUNT>
__device__ __forceinline__ void q_sliced(const QParams &P, int sv, int need, int k, int me, u64 r_lo, u64 ck,
                                         u64 L, const Clauses<M> &cc, const u32 *sw, Work &wk,
                                         const u64 *skj, u64 wstar, i64 &key, i64 &key_m) {
  const int lane = threadIdx.x & 31;
  u64 my_lo = r_lo, my_cnt = (need && r_lo < ck) ? ((ck - r_lo) < L ? (ck - r_lo) : L) : 0ull;
  for (;;) {
    if (my_cnt) {
      int stop = 0;
      i64 km = GR_KEY_NONE;
      const i64 kp = q_walk<M, KIND, COUNT, true>(P, sv, need, k, me, my_lo, my_cnt, cc, sw, 0, wk, skj, wstar,
                                                  &km, (unsigned)clock() + P.slice, &stop);
      key = kp < key ? kp : key;
      key_m = km < key_m ? km : key_m;
      my_lo += (u64)stop;
      my_cnt -= (u64)stop;
    }
    const unsigned busy = __ballot_sync(0xffffffffu, my_cnt != 0);
    if (!busy) break;
    if (busy == 0xffffffffu) continue;
    u64 v = my_cnt;  // the busy lane with the most left gives it out
    int src = lane;
    for (int o = 16; o; o >>= 1) {
      const u64 v2 = __shfl_xor_sync(0xffffffffu, v, o);
      const int s2 = __shfl_xor_sync(0xffffffffu, src, o);
      if (v2 > v || (v2 == v && s2 < src)) { v = v2; src = s2; }
    }
    const u64 dlo = __shfl_sync(0xffffffffu, my_lo, src);
    const int nidle = 32 - __popc(busy);
    if (v < (u64)P.split_min * (u64)(nidle + 1)) continue;
    const u64 part = v / (u64)(nidle + 1);
    if (lane == src) {
      my_cnt = part;
    } else if (!((busy >> lane) & 1u)) {
      const int ir = __popc(~busy & ((1u << lane) - 1u));
      my_lo = dlo + (u64)(ir + 1) * part;
      my_cnt = ir + 1 == nidle ? v - (u64)nidle * part : part;
    }
  }
}

template <bool COUNT, int NTK, int KIND>
__global__ void __launch_bounds__(NTK, COUNT ? 1 : ENUM_CTAS * NT / NTK) queue_kernel(const __grid_constant__ QParams P) {
  extern __shared__ u64 cls[];  // tables, then the staged clause records
  __shared__ int s_b, s_k, s_sv, s_cur, s_exit, s_rb;
  __shared__ u64 s_ti, s_L, s_nch, s_ck;
  __shared__ u64 s_next;  // a next level this CTA committed and keeps (ti + 1 | sv << 40), 0: none
  __shared__ u64 s_skj[JMAX + 1], s_wstar;  // weighted: S_j and the incumbent W*
  __shared__ u32 s_w[64];
  const int t = threadIdx.x, lane = t & 31;
  if (t == 0) s_cur = -1, s_next = 0;
  F2 *hitx = (F2 *)cls;
  u64 *cs = cls + 2 * (JMAX + 1) * HX;
  F2 *lowb = (F2 *)(cs + 65 * (JMAX + 1));
  for (int q = t; q < (JMAX + 1) * HX; q += NTK)
    hitx[q] = F2{g_hit.lo[64 * (q / HX) + q % HX], g_hit.hi[64 * (q / HX) + q % HX]};
  for (int q = t; q < 65 * (JMAX + 1); q += NTK) cs[q] = binom(q / (JMAX + 1), q % (JMAX + 1));
  for (int q = t; q < 129; q += NTK) lowb[q] = f2_nbits((u64)q);
  int *reg = (int *)(lowb + 129);
  if (t <= JMAX) reg[t] = t ? region_of(t) : 0;
  unsigned char *nb = (unsigned char *)(reg + 16);
  for (int q = t; q < (JMAX + 1) * 65; q += NTK) {
    const int jj = q / 65, ee = q % 65;
    nb[q] = jj ? (unsigned char)binom(ee < region_of(jj) ? ee : region_of(jj), jj) : 0;
  }
  u64 *stage = cls + TAB_SMEM / 8;
  for (;;) {
    // ---- thread 0: the small next level this CTA committed, else take a
    // ticket and wait for its ring entry (or the end)
    if (t == 0) {
      Ctrl *ctrl = P.ws[0].ctrl;
      int ex = 0;
      u64 v = 0;
      if (s_next) {
        v = ((s_next >> 40) << 38) | ((s_next & ((1ull << 40) - 1ull)) - 1ull);
        s_next = 0;
      } else {
        const u64 e = atomicAdd((unsigned long long *)&ctrl->q_tickets, 1ull);
        const u64 *r = P.ws[0].ring + (e & P.ring_mask);
        const u64 want = ring_stamp(P, e);
        for (int spin = 0;; spin++) {
          v = ld_acquire(r);  // the task record is read after its entry
          if ((v & ~((1ull << 40) - 1ull)) == want) break;
          if (vld(&ctrl->q_remaining) == 0) { ex = 1; break; }
          __nanosleep(spin < 16 ? 32 : 128);
        }
        if (!ex && (v >> 39 & 1ull)) atomicAdd((unsigned long long *)&ctrl->q_budget, 1ull);  // an extra entry is read
      }
      s_exit = ex;
      if (!ex) {
        const int tsv = (int)((v >> 38) & 1ull);
        const u64 ti = v & ((1ull << 38) - 1ull);
        const Task *T = P.ws[tsv].tasks + ti;
        s_ti = ti;
        s_sv = tsv;
        s_b = T->b;
        s_k = T->k;
        s_L = T->L;
        s_nch = T->nchunks;
        s_rb = T->rb;
        s_ck = binom(P.ws[tsv].meff[s_b], s_k);
      }
    }
    __syncthreads();
    if (s_exit) break;
    {
      const int b = s_b, sv = s_sv;
      const WS &w = P.ws[sv];
      const int np = w.npr[b], nn = w.nnr[b];
      const int64_t lo = P.in[sv].off[b];
      const bool staged = np + nn <= smc_of<NTK>();
      F2 *sH = (F2 *)stage;
      u64 *sP = stage + (size_t)2 * HREC * np;
      const int key_cur = sv * P.in[0].B + b;
      if (key_cur != s_cur) {  // stage the instance's clause records
        if (staged) {
          for (int q = t; q < np * HREC; q += NTK) sH[q] = ((const F2 *)w.hrec)[lo * HREC + q];
          if (w.meff[b] <= 32) {
            u32 *c32 = (u32 *)sP;
            for (int q = t; q < np + nn; q += NTK) c32[q] = (u32)w.pk[lo + q];
          } else {
            for (int q = t; q < np + nn; q += NTK) sP[q] = w.pk[lo + q];
          }
        }
        if (t < 64) s_w[t] = w.wr[(size_t)b * 64 + t];
        if (KIND == 2 && t <= JMAX) s_skj[t] = w.sk[(size_t)b * 65 + t];
      }
      // incumbent of earlier levels (a speculative level may see an older,
      // larger one: it only prunes less)
      if (KIND == 2 && t == 0) s_wstar = vld(&w.bestw[b]);
    }
    __syncthreads();
    if (t == 0) s_cur = s_sv * P.in[0].B + s_b;
    // ---- warps pull warp chunks of this task until it is exhausted.  Lane 0
    // claims one chunk ahead, so the atomic's latency overlaps the walk (not
    // for the weighted walk: the claimed index held across it would spill).
    // The warp whose claim is the first one past the end may publish the next
    // level speculatively, so that idle CTAs work on it while this level's
    // last chunks finish.
    constexpr bool AHEAD = KIND != 2;
    u64 cn = 0;
    if (AHEAD && lane == 0) cn = atomicAdd((unsigned long long *)&P.ws[s_sv].tasks[s_ti].claimed, 1ull);
    for (;;) {
      const int b = s_b, sv = s_sv;
      const u64 nch = s_nch;
      u64 c = AHEAD ? cn : 0ull;
      if (!AHEAD && lane == 0) c = atomicAdd((unsigned long long *)&P.ws[sv].tasks[s_ti].claimed, 1ull);
      int need = 0;  // bit 0: the chunk is needed (fused: for the PMS); bit 1: fused, for the MHS
      if (lane == 0 && c < nch) {
        const Task *T = P.ws[sv].tasks + s_ti;
        const u64 r0 = c * 32 * s_L;
        if (*(const volatile unsigned char *)&T->cancelled) {
          c = nch + 1;  // cancelled speculation: stop claiming
        } else if (KIND == 1) {
          const i64 c1 = vld(&T->key[0]), c2 = vld(&T->key[1]);
          const int np_ = !vld(&P.ws[0].done[b]) && !(c1 != GR_KEY_NONE && (u64)c1 < r0 && !P.exhaustive);
          const int nm_ = !vld(&P.ws[1].done[b]) && !(c2 != GR_KEY_NONE && (u64)c2 < r0 && !P.exhaustive);
          need = np_ | (nm_ << 1);
        } else if (!P.weighted[sv] && !P.exhaustive) {
          const i64 cur = vld(&T->key[0]);
          need = !(cur != GR_KEY_NONE && (u64)cur < r0);  // a lower witness exists
        } else {
          need = 1;
        }
        if (AHEAD && c < nch) cn = atomicAdd((unsigned long long *)&P.ws[sv].tasks[s_ti].claimed, 1ull);
      }
      c = __shfl_sync(0xffffffffu, c, 0);
      if (c >= nch) {
        if (c == nch && lane == 0) P.ws[sv].tasks[s_ti].t_exhaust = gtime();
        if (c == nch && P.spec) {  // the first claim past the end: maybe publish level k+1 now
          u64 n = 0, word = 0, e0 = 0;
          if (lane == 0) {
            Task *T = P.ws[sv].tasks + s_ti;
            const WS &w = P.ws[sv];
            const int k = s_k;
            // only when CTAs are idle (they hold tickets no entry was published
            // for yet): a speculative level never displaces queued work
            const Ctrl *qc = P.ws[0].ctrl;
            const u64 ck1 = binom(w.meff[b], k + 1);
            // ... and only for a level small enough that its chunks in flight
            // cost little if it turns out not to be needed (GR_QSPEC_MAX)
            // (not for weighted levels: the S_k stop rule ends them often)
            if (T->depth < P.spec && !P.weighted[sv] && !*(const volatile unsigned char *)&T->cancelled && k < w.kmax[b] &&
                ck1 <= P.spec_max && vldu(&T->succ) == 0u &&
                (!P.spec_idle || vld(&qc->q_tickets) > vld(&qc->q_entries))) {
              u64 *qw = &w.ctrl->q_work;
              const u64 wk = atomicAdd((unsigned long long *)qw, (unsigned long long)ck1) + ck1;
              u64 ti2;
              bool ok = q_make(P, sv, b, k + 1, wk, T->depth + 1, &ti2);
              if (ok) {
                __threadfence();  // the record before it is linked and published
                ok = atomicCAS(&T->succ, 0u, (unsigned)(ti2 + 1)) == 0u;
              }
              if (ok) {
                word = ti2 | ((u64)sv << 38);
                n = q_entries(P, w.tasks[ti2].nchunks, &e0);
              } else {
                work_sub(qw, ck1);  // level k committed meanwhile (or no room): not needed
              }
            }
          }
          n = __shfl_sync(0xffffffffu, n, 0);
          word = __shfl_sync(0xffffffffu, word, 0);
          e0 = __shfl_sync(0xffffffffu, e0, 0);
          for (u64 i = lane; i < n; i += 32) q_publish(P, word, e0, i);
        }
        break;
      }
      need = __shfl_sync(0xffffffffu, need, 0);
      i64 key = GR_KEY_NONE, key_m = GR_KEY_NONE;
      Work wk;
      {
        const WS &w = P.ws[sv];
        const u64 L = s_L, ck = s_ck;
        const int k = s_k, me = w.meff[b], np = w.npr[b], nn = w.nnr[b];
        const u64 r_lo = c * 32 * L + (u64)lane * L;
        const bool staged = np + nn <= smc_of<NTK>();
        F2 *sH = (F2 *)stage;
        u64 *sP = stage + (size_t)2 * HREC * np;
        if (KIND == 1 && P.slice && staged && me <= 32) {  // (warp-uniform)
          // (not above 32 variables: C3's exhaustive windows are uniformly
          // busy, and slicing them measured 2.44 -> 3.49 ms)
          Clauses<u32> cc{(const u32 *)sP, sH, np, nn};
          q_sliced<u32, KIND, COUNT>(P, sv, need, k, me, r_lo, ck, L, cc, s_w, wk, s_skj, s_wstar, key, key_m);
        } else if (need && r_lo < ck) {
          const u64 cnt = (ck - r_lo) < L ? (ck - r_lo) : L;
          const int64_t lo = P.in[sv].off[b];
          const int rb = KIND == 2 ? s_rb : 0;
          if (staged && me <= 32) {
            Clauses<u32> cc{(const u32 *)sP, sH, np, nn};
            key = q_walk<u32, KIND, COUNT>(P, sv, need, k, me, r_lo, cnt, cc, s_w, rb, wk, s_skj, s_wstar, &key_m);
          } else if (staged) {
            Clauses<u64> cc{sP, sH, np, nn};
            key = q_walk<u64, KIND, COUNT>(P, sv, need, k, me, r_lo, cnt, cc, s_w, rb, wk, s_skj, s_wstar, &key_m);
          } else {
            Clauses<u64> cc{w.pk + lo, (const F2 *)w.hrec + lo * HREC, np, nn};
            key = q_walk<u64, KIND, COUNT>(P, sv, need, k, me, r_lo, cnt, cc, s_w, rb, wk, s_skj, s_wstar, &key_m);
          }
        }
      }
      if (COUNT) work_add(wk, P.ws[s_sv].meff[s_b] > 32);
      key = warp_min(key);
      if (KIND == 1) key_m = warp_min(key_m);
      u64 n = 0, word = 0, e0 = 0;
      if (lane == 0) {
        Task *T = P.ws[s_sv].tasks + s_ti;
        if (key != GR_KEY_NONE) atomicMin((long long *)&T->key[0], (long long)key);
        if (KIND == 1 && key_m != GR_KEY_NONE) atomicMin((long long *)&T->key[1], (long long)key_m);
        // release: the keys before the completion count; acquire: the last
        // arriver sees every chunk's keys
        if (atom_add_acq_rel(&T->pending, ~0ull) == 1ull) {
          // a small next level stays with this CTA: no ring entry, its
          // instance is staged already
          u64 loc = 0;
          n = q_commit_chain(P, s_sv, s_ti, &word, &e0, (u64)P.local_max, &loc);
          if (loc) s_next = loc | ((u64)s_sv << 40);
        }
      }
      n = __shfl_sync(0xffffffffu, n, 0);
      if (n) {  // publish the next level's ring entries together
        word = __shfl_sync(0xffffffffu, word, 0);
        e0 = __shfl_sync(0xffffffffu, e0, 0);
        for (u64 i = lane; i < n; i += 32) q_publish(P, word, e0, i);
      }
    }
    __syncthreads();  // every warp is done with this task's staging
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
int validate_batch(const gr_batch *in, int which) {
  if (!in) { gr_set_error("null batch"); return GR_EINVAL; }
  if (in->B < 1 || (in->W != 1 && in->W != 2)) { gr_set_error("B < 1 or W not in {1,2}"); return GR_EINVAL; }
  if (!in->m || !in->off || !in->n_pos || (!in->masks && in->total_clauses > 0)) {
    gr_set_error("null device pointer in batch");
    return GR_EINVAL;
  }
  if (in->total_clauses < 0 || in->max_clauses < 0) { gr_set_error("negative sizes"); return GR_EINVAL; }
  if (in->max_clauses > MAXC) { gr_set_error("max_clauses > 4096 for the exact solvers"); return GR_ETOOBIG; }
  if (which == 0 && in->w && in->wstride < 1) { gr_set_error("wstride < 1 with weights"); return GR_EINVAL; }
  return GR_OK;
}

template <int NTK>
int enum_grid_of() {
  int per = 0;
  const size_t smem = enum_smem_of<NTK>();
  cudaFuncSetAttribute(enum_kernel<false, NTK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(enum_kernel<true, NTK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, enum_kernel<false, NTK>, NTK, smem);
  return gr_sm_count() * (per < 1 ? 1 : per);
}
// grid of the NT-thread (small = false) or NT/2-thread enumeration CTA, per
// device (the smem attribute is set on each device's first use)
PerDevice g_enum_grid[2];
int enum_grid(bool small = false) {
  return small ? g_enum_grid[1].get(enum_grid_of<NT_SMALL>) : g_enum_grid[0].get(enum_grid_of<NT>);
}
// the small CTA shape when every instance's clauses fit its staging area
bool enum_small(const gr_batch *in) {
  static const int off = getenv("GR_NO_SMALL_CTA") ? 1 : 0;
  return !off && in->max_clauses <= smc_of<NT_SMALL>();
}
template <bool COUNT>
int launch_enum(const EnumParams &p, bool small, cudaStream_t st) {
  if (small)
    GR_LAUNCH("enum_kernel", st, (enum_kernel<COUNT, NT_SMALL><<<enum_grid(true), NT_SMALL,
                                                               enum_smem_of<NT_SMALL>(), st>>>(p)));
  else
    GR_LAUNCH("enum_kernel", st, (enum_kernel<COUNT, NT><<<enum_grid(false), NT, enum_smem_of<NT>(), st>>>(p)));
  return GR_OK;
}

// environment knobs, read once (thread-safe static init)
u64 lane_cands_raw() {
  static const u64 v = [] {
    const char *e = getenv("GR_LANE_CANDIDATES");
    if (!e) return ~0ull;
    u64 x = strtoull(e, nullptr, 10);       // 0: adaptive per level
    return x > (1ull << 20) ? (1ull << 20) : x;  // the walk keeps window positions in 32 bits
  }();
  return v;
}
int windows_per_lane(bool weighted) {  // adaptive lane window: windows per lane per level
  auto rd = [](const char *name, int dflt) {  // GR_WINDOWS_PER_LANE / _W override
    const char *e = getenv(name);
    const int x = e ? atoi(e) : dflt;
    return (x < 1 || x > 0xffff) ? dflt : x;
  };
  static const int v[2] = {rd("GR_WINDOWS_PER_LANE", 3), rd("GR_WINDOWS_PER_LANE_W", 4)};
  return v[weighted ? 1 : 0];
}
u64 lane_max(bool weighted) {  // the adaptive lane window's upper bound
  auto rd = [](const char *name, u64 dflt) {  // GR_LANE_MAX / GR_LANE_MAX_W override
    const char *e = getenv(name);
    u64 x = e ? strtoull(e, nullptr, 10) : dflt;
    if (x > (1ull << 24)) x = 1ull << 24;
    return x < 256 ? dflt : x;
  };
  static const u64 v[2] = {rd("GR_LANE_MAX", 262144ull), rd("GR_LANE_MAX_W", 65536ull)};
  return v[weighted ? 1 : 0];
}
// the device level loop's lane window knobs: GR_QWPL /
// GR_QWPL_W (windows per lane over the work in flight), GR_QLANE_MIN,
// GR_QLANE_MAX / GR_QLANE_MAX_W -- powers of two
u64 env_u64(const char *name, u64 dflt, u64 lo, u64 hi) {
  const char *e = getenv(name);
  const u64 x = e ? strtoull(e, nullptr, 10) : dflt;
  return (x < lo || x > hi) ? dflt : x;
}
struct QKnobs {
  int wpl, wpl_w;
  u64 lmin, lmax, lmax_w, lmin_w;
};
const QKnobs &qknobs() {
  static const QKnobs k = {(int)env_u64("GR_QWPL", 1, 1, 0xffff), (int)env_u64("GR_QWPL_W", 1, 1, 0xffff),
                           env_u64("GR_QLANE_MIN", 4096, 1, 1ull << 20),
                           env_u64("GR_QLANE_MAX", 1ull << 20, 256, 1ull << 24),
                           env_u64("GR_QLANE_MAX_W", 1ull << 16, 256, 1ull << 24),
                           env_u64("GR_QLANE_MIN_W", 2048, 1, 1ull << 20)};
  return k;
}
u64 lane_cands() {  // 0 = adaptive (GR_LANE_CANDIDATES overrides)
  const u64 v = lane_cands_raw();
  return v == ~0ull ? 0ull : v;
}

}  // namespace

extern "C" size_t gr_workspace_bytes_exact(const gr_batch *in) { return layout_of(in).total; }

// diagnostics (scripts/queue_stats.py): byte offset of the task records in a
// workspace of gr_workspace_bytes(in, 0)
extern "C" size_t gr_debug_tasks_offset(const gr_batch *in) { return layout_of(in).tasks; }

// per-instance u64 scratch of the exact workspace that no solve touches
// (gr_solve keeps the greedy costs there across the final MaxSAT query)
uint64_t *gr_exact_scratch(const gr_batch *in, void *ws) {
  return (uint64_t *)((char *)ws + layout_of(in).gcost);
}

void gr_exact_work_read(unsigned long long out[8], int reset) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { for (int i = 0; i < W_N; i++) out[i] = 0; return; }
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out, g_work, sizeof(unsigned long long) * W_N) != cudaSuccess)
    for (int i = 0; i < W_N; i++) out[i] = 0;
  if (reset) {
    unsigned long long z[W_N] = {};
    cudaMemcpyToSymbol(g_work, z, sizeof(z));
  }
}

namespace {
int *pinned_i32() {
  static thread_local int *p = nullptr;
  if (!p) {
    if (cudaMallocHost((void **)&p, 64) != cudaSuccess) p = nullptr;
  }
  return p;
}
}  // namespace

namespace {
int launch_finish(const gr_batch *in, int which, const gr_result *out, const WS &w, int k,
                  cudaStream_t st, const int *done_other) {
  const int fgrid = k > 0 ? std::max(1, std::min((in->B + FT - 1) / FT, 64)) : 1;
  GR_LAUNCH("finish_kernel", st, finish_kernel<<<fgrid, FT, 0, st>>>(in_of(in, which), out_of(out), w, which, k,
                                   (in->flags & GR_FLAG_EXHAUSTIVE) ? 1 : 0, enum_grid() * NT, lane_cands(), windows_per_lane(false) | (windows_per_lane(true) << 16),
                                   lane_max(false), lane_max(true), done_other,
                                   enum_small(in) ? NT_SMALL : NT));
  return GR_OK;
}
// pack the batch for one solve, or for two (which1 >= 0: the second solve's
// result and workspace) in the same launch
int launch_pack(const gr_batch *in, int which, const gr_result *out, const WS &w, cudaStream_t st,
                int which1 = -1, const gr_result *out1 = nullptr, const WS *w1 = nullptr) {
  PackArgs A{};
  A.in[0] = in_of(in, which);
  A.out[0] = out_of(out);
  A.ws[0] = w;
  A.which[0] = which;
  const int two = which1 >= 0 ? 1 : 0;
  A.in[1] = two ? in_of(in, which1) : A.in[0];
  A.out[1] = two ? out_of(out1) : A.out[0];
  A.ws[1] = two ? *w1 : w;
  A.which[1] = two ? which1 : which;
  A.lane_cands = lane_cands();
  A.ring_n = ring_cap(in->B);
  size_t smem = (size_t)std::max(in->max_clauses, 1) * 13 + 16;
  static PerDevice attr;
  attr.get([] { return (int)cudaFuncSetAttribute(pack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, MAXC * 13 + 16); });
  GR_LAUNCH("pack_kernel", st, pack_kernel<<<in->B * (1 + two), PT, smem, st>>>(A));
  return GR_OK;
}
}  // namespace

extern "C" int gr_exact_prepare(const gr_batch *in, int which, gr_result *out, void *ws,
                                size_t ws_bytes, gr_stream_t s, int32_t *n_active) {
  int rc = validate_batch(in, which);
  if (rc) return rc;
  if (!out || !out->assign || !out->cost || !out->status) { gr_set_error("null result pointer"); return GR_EINVAL; }
  if (which != 0 && which != 1) { gr_set_error("which must be 0 (PMS) or 1 (MHS)"); return GR_EINVAL; }
  Layout L = layout_of(in);
  if (!ws || ws_bytes < L.total) { gr_set_error("workspace too small"); return GR_EWORKSPACE; }
  WS w = ws_of(in, ws);
  cudaStream_t st = (cudaStream_t)s;
  if ((rc = launch_pack(in, which, out, w, st))) return rc;
  if ((rc = launch_finish(in, which, out, w, 0, st, nullptr))) return rc;
  if (n_active) {
    int *h = pinned_i32();
    if (!h) { gr_set_error("cudaMallocHost failed"); return GR_ECUDA; }
    GR_CUDA(cudaMemcpyAsync(h, &w.ctrl->n_remaining, sizeof(int), cudaMemcpyDeviceToHost, st));
    GR_CUDA(cudaStreamSynchronize(st));
    *n_active = *h;
  }
  return GR_OK;
}

extern "C" int gr_exact_level(const gr_batch *in, int which, int k, int shard, int nshard, void *ws,
                              size_t ws_bytes, gr_stream_t s) {
  int rc = validate_batch(in, which);
  if (rc) return rc;
  if (k < 1 || k > 64 || nshard < 1 || shard < 0 || shard >= nshard) { gr_set_error("bad level/shard"); return GR_EINVAL; }
  Layout L = layout_of(in);
  if (!ws || ws_bytes < L.total) { gr_set_error("workspace too small"); return GR_EWORKSPACE; }
  WS w = ws_of(in, ws);
  // the list of level k lives at parity k & 1
  w.active = w.active + (size_t)(k & 1) * in->B;
  EnumParams p;
  p.ws = w;
  p.off = in->off;
  p.k = k;
  p.weighted = (which == 0 && in->w) ? 1 : 0;
  p.exhaustive = (in->flags & GR_FLAG_EXHAUSTIVE) ? 1 : 0;
  p.prune = (in->flags & GR_FLAG_NO_PRUNE) ? 0 : 1;
  p.shard = shard;
  p.nshard = nshard;
  p.fused = 0;
  p.ws2 = w;
  int grid = enum_grid();
  // the finish kernel leaves next_chunk at 0; several shards of one level on
  // one device (multi-shard emulation) need it reset between them
  if (nshard > 1) GR_CUDA(cudaMemsetAsync(&w.ctrl->next_chunk, 0, sizeof(u64), (cudaStream_t)s));
  (void)grid;
  return gr_prof_mode() == 2 ? launch_enum<true>(p, enum_small(in), (cudaStream_t)s)
                             : launch_enum<false>(p, enum_small(in), (cudaStream_t)s);
}

extern "C" int64_t *gr_exact_level_keys(const gr_batch *in, int which, void *ws) {
  (void)which;
  if (!in || !ws) return nullptr;
  return (int64_t *)ws_of(in, ws).lvlkey;
}

extern "C" int gr_exact_finish(const gr_batch *in, int which, int k, gr_result *out, void *ws,
                               size_t ws_bytes, gr_stream_t s, int32_t *n_active) {
  int rc = validate_batch(in, which);
  if (rc) return rc;
  Layout L = layout_of(in);
  if (!ws || ws_bytes < L.total) { gr_set_error("workspace too small"); return GR_EWORKSPACE; }
  if (k < 1 || k > 64) { gr_set_error("bad level"); return GR_EINVAL; }
  WS w = ws_of(in, ws);
  cudaStream_t st = (cudaStream_t)s;
  const int fgrid = std::max(1, std::min((in->B + FT - 1) / FT, 64));
  GR_LAUNCH("finish_kernel", (cudaStream_t)s, finish_kernel<<<fgrid, FT, 0, st>>>(in_of(in, which), out_of(out), w, which, k,
                                   (in->flags & GR_FLAG_EXHAUSTIVE) ? 1 : 0, enum_grid() * NT, lane_cands(), windows_per_lane(false) | (windows_per_lane(true) << 16),
                                   lane_max(false), lane_max(true), nullptr,
                                   enum_small(in) ? NT_SMALL : NT));
  if (n_active) {
    int *h = pinned_i32();
    if (!h) { gr_set_error("cudaMallocHost failed"); return GR_ECUDA; }
    GR_CUDA(cudaMemcpyAsync(h, &w.ctrl->n_remaining, sizeof(int), cudaMemcpyDeviceToHost, st));
    GR_CUDA(cudaStreamSynchronize(st));
    *n_active = *h;
  }
  return GR_OK;
}

// s_other waits for the work queued on st so far (results ordered on both)
static int stream_join(cudaStream_t st, cudaStream_t s_other) {
  if (s_other == st) return GR_OK;
  cudaEvent_t ev;
  GR_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  GR_CUDA(cudaEventRecord(ev, st));
  GR_CUDA(cudaStreamWaitEvent(s_other, ev, 0));
  GR_CUDA(cudaEventDestroy(ev));
  return GR_OK;
}

// levels queued per host read-back of n_active (GR_SPEC_LEVELS)
static int spec_levels() {
  static const int v = [] {
    const char *e = getenv("GR_SPEC_LEVELS");
    const int x = e ? atoi(e) : 4;
    return (x < 1 || x > 64) ? 4 : x;
  }();
  return v;
}

// ---- the device level loop (queue_kernel) ------------------------------------
namespace {
std::atomic<unsigned long long> g_qgen{0};
template <int NTK, int KIND>
void queue_attr() {
  const int smem = (int)enum_smem_of<NTK>();
  cudaFuncSetAttribute(queue_kernel<false, NTK, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(queue_kernel<true, NTK, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}
template <int NTK>
int queue_grid_of() {
  int per = 0;
  queue_attr<NTK, 0>();
  queue_attr<NTK, 1>();
  queue_attr<NTK, 2>();
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, queue_kernel<false, NTK, 0>, NTK, enum_smem_of<NTK>());
  return gr_sm_count() * (per < 1 ? 1 : per);
}
PerDevice g_queue_grid[2];
int queue_grid(bool small) {
  return small ? g_queue_grid[1].get(queue_grid_of<NT_SMALL>) : g_queue_grid[0].get(queue_grid_of<NT>);
}
// GR_HOST_LOOP=1: the level-synchronous host loop (enum + finish launches per
// level) instead of queue_kernel -- A/B timing and cross-checks only
bool host_loop() {
  static const bool v = getenv("GR_HOST_LOOP") != nullptr;
  return v;
}

template <bool COUNT, int NTK, int KIND>
int launch_queue_t(QParams &P, int B, cudaStream_t st) {
  const int grid = queue_grid(NTK == NT_SMALL);
  P.grid = grid;
  P.nwarps = NTK / 32;
  if (P.local_max > P.nwarps) P.local_max = P.nwarps;
  P.lanes = grid * NTK;
  // extra ring entries beyond one per open unit and the tickets the grid holds
  const long long budget = (long long)ring_cap(B) - (long long)(P.fused ? 1 : P.nsolve) * B -
                           2ll * grid - 64;
  const int sg = std::max(1, std::min((B + 255) / 256, 4 * gr_sm_count()));
  GR_LAUNCH("queue_work_kernel", st, queue_work_kernel<<<sg, 256, 0, st>>>(P, budget));
  GR_LAUNCH("queue_seed_kernel", st, queue_seed_kernel<<<sg, 256, 0, st>>>(P));
  GR_LAUNCH("queue_kernel", st, (queue_kernel<COUNT, NTK, KIND><<<grid, NTK, enum_smem_of<NTK>(), st>>>(P)));
  return GR_OK;
}

// one launch for the level loops of one solve (nsolve = 1), of two
// independent solves of the same batch (nsolve = 2: weighted PMS + MHS), or
// of the fused PMS + MHS walk (fused = 1); the packs already ran on st
int launch_queue(const gr_batch *in, int nsolve, int fused, const int which[2], gr_result *o0,
                 gr_result *o1, const WS &w0, const WS &w1, cudaStream_t st) {
  QParams P{};
  P.ws[0] = w0;
  P.ws[1] = w1;
  P.in[0] = in_of(in, which[0]);
  P.in[1] = in_of(in, which[1]);
  P.out[0] = out_of(o0);
  P.out[1] = out_of(o1 ? o1 : o0);
  for (int q = 0; q < 2; q++) {
    P.which[q] = which[q];
    P.weighted[q] = (!fused && P.in[q].w != nullptr) ? 1 : 0;
  }
  P.nsolve = nsolve;
  P.fused = fused;
  P.exhaustive = (in->flags & GR_FLAG_EXHAUSTIVE) ? 1 : 0;
  P.prune = (in->flags & GR_FLAG_NO_PRUNE) ? 0 : 1;
  P.spec = (int)env_u64("GR_QSPEC", 2, 0, 16);  // speculative levels ahead (0: off)
  P.spec_max = env_u64("GR_QSPEC_MAX", 1ull << 32, 0, ~0ull);
  P.gen = g_qgen.fetch_add(1) % 4095ull + 1ull;  // 1..4095
  P.ring_mask = ring_cap(in->B) - 1;
  P.ring_log2 = 63 - __builtin_clzll(ring_cap(in->B));
  const QKnobs &kn = qknobs();
  P.wpl = kn.wpl | (kn.wpl_w << 16);
  P.lane_max = kn.lmax;
  P.lane_max_w = kn.lmax_w;
  P.fixed_lane = lane_cands();
  P.lane_min = kn.lmin | (kn.lmin_w << 32);
  static const int ql = (int)env_u64("GR_QLOCAL", 1, 0, 1ull << 30);  // (capped at the warps per CTA)
  P.local_max = ql;
  static const u64 qs = env_u64("GR_QLANE_SPLIT", 1ull << 62, 1, 1ull << 62);  // default: off
  P.lane_split = qs;
  // speculation waits for idle CTAs, except in the fused walk (C2: its
  // heavy instances' level chains are the critical path; measured 0.637 ->
  // 0.61 ms); GR_QSPEC_IDLE=0|1 forces either
  static const int qsi = (int)env_u64("GR_QSPEC_IDLE", 2, 0, 2);
  P.spec_idle = qsi == 2 ? (fused ? 0 : 1) : qsi;
  // fused walk time slice: 10^5 clocks (~51 us); the heavy windows of C2's
  // critical instance are then shared by their warps' idle lanes
  // (C2 0.61 -> 0.575 ms; 0: untimed)
  static const unsigned qsl = (unsigned)env_u64("GR_QSLICE", 100000, 0, 1u << 30);
  static const int qsm = (int)env_u64("GR_QSPLIT_MIN", 256, 1, 1u << 30);
  P.slice = qsl;
  P.split_min = qsm;
  const bool small = enum_small(in);
  const int kind = fused ? 1 : ((P.weighted[0] || P.weighted[1]) ? 2 : 0);
#define GR_QLAUNCH(COUNT, NTK)                                              \
  return kind == 0 ? launch_queue_t<COUNT, NTK, 0>(P, in->B, st)            \
         : kind == 1 ? launch_queue_t<COUNT, NTK, 1>(P, in->B, st)          \
                     : launch_queue_t<COUNT, NTK, 2>(P, in->B, st)
  if (gr_prof_mode() == 2) {
    if (small) GR_QLAUNCH(true, NT_SMALL);
    GR_QLAUNCH(true, NT);
  }
  if (small) GR_QLAUNCH(false, NT_SMALL);
  GR_QLAUNCH(false, NT);
#undef GR_QLAUNCH
}
}  // namespace

static int solve_exact(const gr_batch *in, gr_result *out, void *ws, size_t ws_bytes, gr_stream_t s,
                       int which) {
  if (!host_loop()) {
    int rc = validate_batch(in, which);
    if (rc) return rc;
    if (!out || !out->assign || !out->cost || !out->status) { gr_set_error("null result pointer"); return GR_EINVAL; }
    Layout L = layout_of(in);
    if (!ws || ws_bytes < L.total) { gr_set_error("workspace too small"); return GR_EWORKSPACE; }
    WS w = ws_of(in, ws);
    cudaStream_t st = (cudaStream_t)s;
    if ((rc = launch_pack(in, which, out, w, st))) return rc;
    const int wh[2] = {which, which};
    return launch_queue(in, 1, 0, wh, out, nullptr, w, w, st);
  }
  int32_t n = 0;  // level 0 is handled by the pack; instances active for level 1
  int rc = gr_exact_prepare(in, which, out, ws, ws_bytes, s, &n);
  if (rc) return rc;
  // levels are queued SPEC at a time and n_active is read back once per batch;
  // levels past the last active one are no-ops (empty active list)
  const int SPEC = spec_levels();
  for (int k = 1; n > 0 && k <= 64;) {
    for (int i = 0; i < SPEC && k <= 64; i++, k++) {
      rc = gr_exact_level(in, which, k, 0, 1, ws, ws_bytes, s);
      if (rc) return rc;
      const bool last = i == SPEC - 1 || k == 64;
      rc = gr_exact_finish(in, which, k, out, ws, ws_bytes, s, last ? &n : nullptr);
      if (rc) return rc;
    }
  }
  return GR_OK;
}

int gr_exact_solve_selected(const gr_batch *in, gr_result *out, void *ws, size_t ws_bytes,
                            gr_stream_t s, const int32_t *sel, int sel_val) {
  t_sel = sel;
  t_sel_val = sel_val;
  const int rc = solve_exact(in, out, ws, ws_bytes, s, 0);
  t_sel = nullptr;
  return rc;
}

extern "C" int gr_solve_pms(const gr_batch *in, gr_result *out, void *ws, size_t ws_bytes,
                            gr_stream_t s) {
  return solve_exact(in, out, ws, ws_bytes, s, 0);
}

// ---- fused PMS + MHS step-wise: the pair session (rank-range sharding) ------
// The fused walk (MODE 3) with the level loop owned by the caller, as the
// gr_exact_prepare / level / finish session: ws = two halves of
// gr_workspace_bytes (PMS, then MHS); unit weights only.
static int pair_ws(const gr_batch *in, void *ws, size_t ws_bytes, WS &w1, WS &w2) {
  int rc = validate_batch(in, 0);
  if (rc) return rc;
  if (in->w || in->k_start) { gr_set_error("the fused pair session needs unit weights and no k_start"); return GR_EINVAL; }
  const size_t half = align256(layout_of(in).total);
  if (!ws || ws_bytes < 2 * half) { gr_set_error("workspace too small (2 x gr_workspace_bytes)"); return GR_EWORKSPACE; }
  w1 = ws_of(in, ws);
  w2 = ws_of(in, (char *)ws + half);
  return GR_OK;
}

extern "C" int gr_pair_prepare(const gr_batch *in, gr_result *out_pms, gr_result *out_mhs, void *ws,
                               size_t ws_bytes, gr_stream_t s, int32_t *n_active) {
  WS w1, w2;
  int rc = pair_ws(in, ws, ws_bytes, w1, w2);
  if (rc) return rc;
  if (!out_pms || !out_mhs || !out_pms->assign || !out_mhs->assign) { gr_set_error("null result"); return GR_EINVAL; }
  cudaStream_t st = (cudaStream_t)s;
  if ((rc = launch_pack(in, 1, out_mhs, w2, st))) return rc;
  if ((rc = launch_finish(in, 1, out_mhs, w2, 0, st, nullptr))) return rc;
  if ((rc = launch_pack(in, 0, out_pms, w1, st))) return rc;
  if ((rc = launch_finish(in, 0, out_pms, w1, 0, st, w2.done))) return rc;
  if (n_active) {
    int *h = pinned_i32();
    if (!h) { gr_set_error("cudaMallocHost failed"); return GR_ECUDA; }
    GR_CUDA(cudaMemcpyAsync(h, &w1.ctrl->n_remaining, sizeof(int), cudaMemcpyDeviceToHost, st));
    GR_CUDA(cudaStreamSynchronize(st));
    *n_active = *h;
  }
  return GR_OK;
}

extern "C" int gr_pair_level(const gr_batch *in, int k, int shard, int nshard, void *ws,
                             size_t ws_bytes, gr_stream_t s) {
  WS w1, w2;
  int rc = pair_ws(in, ws, ws_bytes, w1, w2);
  if (rc) return rc;
  if (k < 1 || k > 64 || nshard < 1 || shard < 0 || shard >= nshard) { gr_set_error("bad level/shard"); return GR_EINVAL; }
  cudaStream_t st = (cudaStream_t)s;
  EnumParams p;
  p.ws = w1;
  p.ws.active = w1.active + (size_t)(k & 1) * in->B;
  p.ws2 = w2;
  p.off = in->off;
  p.k = k;
  p.weighted = 0;
  p.exhaustive = (in->flags & GR_FLAG_EXHAUSTIVE) ? 1 : 0;
  p.prune = (in->flags & GR_FLAG_NO_PRUNE) ? 0 : 1;
  p.shard = shard;
  p.nshard = nshard;
  p.fused = 1;
  if (nshard > 1) GR_CUDA(cudaMemsetAsync(&w1.ctrl->next_chunk, 0, sizeof(u64), st));
  return gr_prof_mode() == 2 ? launch_enum<true>(p, enum_small(in), st) : launch_enum<false>(p, enum_small(in), st);
}

extern "C" int64_t *gr_pair_level_keys(const gr_batch *in, void *ws, int which) {
  if (!in || !ws || (which != 0 && which != 1)) return nullptr;
  const size_t half = align256(layout_of(in).total);
  return (int64_t *)ws_of(in, (char *)ws + (which ? half : 0)).lvlkey;
}

extern "C" int gr_pair_finish(const gr_batch *in, int k, gr_result *out_pms, gr_result *out_mhs,
                              void *ws, size_t ws_bytes, gr_stream_t s, int32_t *n_active) {
  WS w1, w2;
  int rc = pair_ws(in, ws, ws_bytes, w1, w2);
  if (rc) return rc;
  if (k < 1 || k > 64) { gr_set_error("bad level"); return GR_EINVAL; }
  if (!out_pms || !out_mhs) { gr_set_error("null result"); return GR_EINVAL; }
  cudaStream_t st = (cudaStream_t)s;
  const int P = std::max(1, std::min((in->B + FT - 1) / FT, 32));
  GR_LAUNCH("finish_kernel", st, finish_fused_kernel<<<2 * P, FT, 0, st>>>(
                                     in_of(in, 0), out_of(out_pms), w1, in_of(in, 1), out_of(out_mhs), w2, k,
                                     (in->flags & GR_FLAG_EXHAUSTIVE) ? 1 : 0, enum_grid() * NT, lane_cands(),
                                     windows_per_lane(false) | (windows_per_lane(true) << 16),
                                     lane_max(false), lane_max(true), enum_small(in) ? NT_SMALL : NT));
  if (n_active) {
    int *h = pinned_i32();
    if (!h) { gr_set_error("cudaMallocHost failed"); return GR_ECUDA; }
    GR_CUDA(cudaMemcpyAsync(h, &w1.ctrl->n_remaining, sizeof(int), cudaMemcpyDeviceToHost, st));
    GR_CUDA(cudaStreamSynchronize(st));
    *n_active = *h;
  }
  return GR_OK;
}

// PMS and MHS of one batch: unit weights -> one fused walk (MODE 3) on s_pms;
// otherwise their level loops interleaved on two streams (the small levels
// and level tails of one overlap the other's work).
extern "C" int gr_solve_pms_mhs(const gr_batch *in, gr_result *out_pms, gr_result *out_mhs,
                                void *ws, size_t ws_bytes, gr_stream_t s_pms, gr_stream_t s_mhs) {
  int rc = validate_batch(in, 0);
  if (rc) return rc;
  const size_t half = align256(layout_of(in).total);
  if (!ws || ws_bytes < 2 * half) { gr_set_error("workspace too small (2 x gr_workspace_bytes)"); return GR_EWORKSPACE; }
  void *ws1 = ws, *ws2 = (char *)ws + half;
  if (!in->w && !in->k_start && !getenv("GR_NO_FUSE")) {
    // unit weights: one walk decides both -- the MHS is phi+'s part of the
    // PMS test (MODE 3); the PMS workspace plans the union of both searches
    if (!out_pms || !out_mhs) { gr_set_error("null result"); return GR_EINVAL; }
    cudaStream_t st = (cudaStream_t)s_pms;
    WS w1 = ws_of(in, ws1), w2 = ws_of(in, ws2);
    if (!host_loop()) {  // both packs in one launch, then one device level loop for the fused walk
      if ((rc = launch_pack(in, 0, out_pms, w1, st, 1, out_mhs, &w2))) return rc;
      const int wh[2] = {0, 1};
      if ((rc = launch_queue(in, 1, 1, wh, out_pms, out_mhs, w1, w2, st))) return rc;
      return stream_join(st, (cudaStream_t)s_mhs);
    }
    // the level-synchronous host loop over the pair session (A/B, GR_HOST_LOOP)
    int32_t n = 0;
    if ((rc = gr_pair_prepare(in, out_pms, out_mhs, ws, ws_bytes, s_pms, &n))) return rc;
    const int SPEC = spec_levels();
    for (int k = 1; n > 0 && k <= 64;) {
      for (int i = 0; i < SPEC && k <= 64; i++, k++) {
        if ((rc = gr_pair_level(in, k, 0, 1, ws, ws_bytes, s_pms))) return rc;
        const bool last = i == SPEC - 1 || k == 64;
        if ((rc = gr_pair_finish(in, k, out_pms, out_mhs, ws, ws_bytes, s_pms, last ? &n : nullptr)))
          return rc;
      }
    }
    return stream_join(st, (cudaStream_t)s_mhs);
  }
  if (!host_loop()) {  // weighted PMS + MHS (or start levels): one launch serves both solves
    if (!out_pms || !out_mhs) { gr_set_error("null result"); return GR_EINVAL; }
    cudaStream_t st = (cudaStream_t)s_pms;
    WS w1 = ws_of(in, ws1), w2 = ws_of(in, ws2);
    if ((rc = launch_pack(in, 0, out_pms, w1, st, 1, out_mhs, &w2))) return rc;
    const int wh[2] = {0, 1};
    if ((rc = launch_queue(in, 2, 0, wh, out_pms, out_mhs, w1, w2, st))) return rc;
    return stream_join(st, (cudaStream_t)s_mhs);
  }
  int32_t n1 = 0, n2 = 0;
  rc = gr_exact_prepare(in, 0, out_pms, ws1, half, s_pms, nullptr);
  if (rc) return rc;
  rc = gr_exact_prepare(in, 1, out_mhs, ws2, half, s_mhs, nullptr);
  if (rc) return rc;
  int *h = pinned_i32();
  if (!h) { gr_set_error("cudaMallocHost failed"); return GR_ECUDA; }
  cudaStream_t st1 = (cudaStream_t)s_pms, st2 = (cudaStream_t)s_mhs;
  WS w1 = ws_of(in, ws1), w2 = ws_of(in, ws2);
  GR_CUDA(cudaMemcpyAsync(h, &w1.ctrl->n_remaining, sizeof(int), cudaMemcpyDeviceToHost, st1));
  GR_CUDA(cudaMemcpyAsync(h + 1, &w2.ctrl->n_remaining, sizeof(int), cudaMemcpyDeviceToHost, st2));
  GR_CUDA(cudaStreamSynchronize(st1));
  GR_CUDA(cudaStreamSynchronize(st2));
  n1 = h[0];
  n2 = h[1];
  const int SPEC = spec_levels();
  for (int k = 1; (n1 > 0 || n2 > 0) && k <= 64;) {
    const bool a1 = n1 > 0, a2 = n2 > 0;
    for (int i = 0; i < SPEC && k <= 64; i++, k++) {
      if (a1) {
        if ((rc = gr_exact_level(in, 0, k, 0, 1, ws1, half, s_pms))) return rc;
        if ((rc = gr_exact_finish(in, 0, k, out_pms, ws1, half, s_pms, nullptr))) return rc;
      }
      if (a2) {
        if ((rc = gr_exact_level(in, 1, k, 0, 1, ws2, half, s_mhs))) return rc;
        if ((rc = gr_exact_finish(in, 1, k, out_mhs, ws2, half, s_mhs, nullptr))) return rc;
      }
    }
    if (a1) GR_CUDA(cudaMemcpyAsync(h, &w1.ctrl->n_remaining, sizeof(int), cudaMemcpyDeviceToHost, st1));
    if (a2) GR_CUDA(cudaMemcpyAsync(h + 1, &w2.ctrl->n_remaining, sizeof(int), cudaMemcpyDeviceToHost, st2));
    if (a1) { GR_CUDA(cudaStreamSynchronize(st1)); n1 = h[0]; }
    if (a2) { GR_CUDA(cudaStreamSynchronize(st2)); n2 = h[1]; }
  }
  return GR_OK;
}

extern "C" int gr_mhs_exact(const gr_batch *in, gr_result *out, void *ws, size_t ws_bytes,
                            gr_stream_t s) {
  return solve_exact(in, out, ws, ws_bytes, s, 1);
}
