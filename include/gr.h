/*
 * gr.h -- C-ABI of libgrsolve.so: the Solve step of GPURepair (arXiv
 * 2011.08373) on NVIDIA B200 (sm_100a).
 *
 * The Solve step (Alg. 1 line `solve`, Alg:gpurepair) takes the
 * constraint phi over the barrier variables b_1..b_m -- positive
 * monotone clauses phi+ from data-race traces and negative monotone clauses
 * phi- from barrier-divergence traces -- and returns an
 * assignment <res, sol> that enables as few barriers as possible, or UNSAT
 * (PAPER.md:131-133).  Three solvers are exported:
 *
 *   gr_solve_pms   exact (weighted) partial MaxSAT: phi hard, {not b_i} soft
 *                  (MaxSAT strategy; PMS/WPMS)
 *   gr_mhs_exact   exact Minimum-Hitting-Set of phi+ 
 *   gr_mhs_greedy  Johnson's greedy minimal hitting set of phi+ (mhs
 *                  strategy), pruned to a *minimal* set
 *                  (reading R12), phi- checked
 *   gr_mhs_greedy_matrix   the same greedy for one huge phi+ stored as a
 *                  variable x clause bit matrix in HBM
 *
 * Conventions (all calls):
 *   - Encoding (reading R1): b_i <-> bit (i-1) of a clause mask; a mask is W
 *     little-endian uint64 words (b_1 = LSB of word 0).  Polarity is
 *     positional: the first n_pos[b] clauses of instance b are positive.
 *   - Pointers inside gr_batch / gr_result / gr_bitmatrix are DEVICE
 *     pointers unless marked "host"; the caller owns every buffer.  The
 *     library allocates no device memory per call: scratch comes from the
 *     caller's workspace (size from gr_*_workspace_bytes, 256-byte aligned).
 *   - Stream-ordered on `s`.  Calls that run a level / iteration loop on the
 *     host (gr_solve_pms, gr_mhs_exact, gr_exact_finish,
 *     gr_mhs_greedy_matrix) synchronise `s` for a few bytes of control state
 *     per level / per 8 iterations; every result is valid once they return.
 *   - Return value: GR_OK or a negative call-level error (nothing is
 *     written to outputs then); per-instance outcomes go to `status`.
 *     UNSAT is a result, not an error.  gr_last_error() describes the last
 *     negative return of the calling thread.
 *   - Re-entrant for distinct workspaces / streams.
 *   - Canonical answers (readings R2, R3, R11): exact solvers return the
 *     optimum with the smallest colex rank (= numerically smallest mask
 *     among optimal sets); WPMS minimises (W, k, mask) lexicographically;
 *     greedy takes the lowest variable index on count ties.
 */
#ifndef GR_H
#define GR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *gr_stream_t; /* a cudaStream_t; NULL = legacy default stream */

/* call-level return codes */
enum {
  GR_OK = 0,
  GR_EINVAL = -1,      /* null pointer, B < 1, W not in {1,2}, bad flags ... */
  GR_ETOOBIG = -2,     /* a size beyond what the build supports (see each call) */
  GR_ECUDA = -3,       /* a CUDA runtime error (gr_last_error has the text) */
  GR_ENOMEM = -4,      /* reserved */
  GR_EWORKSPACE = -5   /* ws == NULL or ws_bytes < the queried size */
};

/* per-instance status */
enum {
  GR_SAT = 0,
  GR_UNSAT = 1,              /* no assignment satisfies the hard clauses (R6, R16) */
  GR_SAT_NEG_VIOLATED = 2,   /* mhs / MHS hits phi+ but some N in phi- has N subset of S:
                                the caller falls back to MaxSAT */
  GR_BADINPUT = 3,           /* a bit >= m is set (R8), a weight is 0 (R4), or the
                                instance exceeds max_clauses */
  GR_UNSUPPORTED = 4         /* exact solvers: |support(phi+)| > 64, or a weighted
                                key (W, rank) that does not fit 63 bits */
};

/* flags of gr_batch.flags */
enum {
  GR_FLAG_EXHAUSTIVE = 1,    /* exact unit-weight solvers: enumerate the witness level
                                completely (deterministic work; benchmarking mode).
                                Results are identical. */
  GR_FLAG_WEIGHTED_GREEDY = 2, /* gr_mhs_greedy / gr_solve(MHS) with w != NULL: the weighted
                                mhs -- pick the variable
                                maximising uncovered-hits / weight (exact cross-multiplied
                                comparison, lowest index on ties, reading R20); cost = weight */
  GR_FLAG_NO_PRUNE = 4       /* exact solvers: decide every sub-block by its clause tests,
                                without refuting whole subtrees first (measurement mode;
                                results and decided counts are identical) */
};

/* A batch of independent Solve-step instances. */
typedef struct {
  int32_t B;                /* host: number of instances, >= 1 */
  int32_t W;                /* host: uint64 words per clause mask, 1 (m <= 64) or 2 (m <= 128) */
  int64_t total_clauses;    /* host: off[B] (sizes the workspace) */
  int32_t max_clauses;      /* host: upper bound on off[b+1]-off[b]; <= 4096 for the exact
                               solvers and for gr_mhs_greedy */
  uint32_t flags;           /* host: GR_FLAG_* */
  const int32_t *m;         /* [B] number of barrier variables, 0 <= m[b] <= 64*W */
  const int64_t *off;       /* [B+1] instance b owns clauses off[b] .. off[b+1]-1 */
  const int32_t *n_pos;     /* [B] the first n_pos[b] clauses of b are positive (phi+) */
  const uint64_t *masks;    /* [off[B]][W] clause masks */
  const uint32_t *w;        /* [B][wstride] weight w_i >= 1 of soft clause (not b_i), i < m[b];
                               NULL = unit weights (PMS).  Read by gr_solve_pms only. */
  int32_t wstride;          /* host: row stride of w in elements (>= max m) */
  const int32_t *k_start;   /* [B] or NULL (incremental Solve): unit-weight
                               exact solvers enumerate levels k >= k_start[b] only.  The caller
                               guarantees that no feasible set has fewer than k_start[b]
                               elements -- e.g. phi grew by clauses since a solve whose optimum
                               had k_start[b] elements (phi := phi U {c} only
                               shrinks the feasible sets).  decided counts enumerated levels.
                               Ignored by WPMS (a lighter optimum may use fewer elements). */
} gr_batch;

/* Per-instance results (device buffers, written by the library). */
typedef struct {
  uint64_t *assign;   /* [B][W] total assignment, bit i-1 = b_i true; 0 when UNSAT/BADINPUT */
  uint64_t *cost;     /* [B] sum of w_i over true b_i (popcount if unit); UINT64_MAX if UNSAT */
  int32_t *status;    /* [B] GR_SAT | GR_UNSAT | GR_SAT_NEG_VIOLATED | GR_BADINPUT | GR_UNSUPPORTED */
  uint64_t *decided;  /* [B] or NULL: candidate assignments whose feasibility was decided
                         (exact solvers; DESIGN.md §5 defines the count) */
} gr_result;

/* Workspace bytes for a call on `in`: which = 0 gr_solve_pms, 1 gr_mhs_exact,
 * 2 gr_mhs_greedy.  Returns 0 on invalid input. */
size_t gr_workspace_bytes(const gr_batch *in, int which);

/* (a) Exact PMS / WPMS: minimise the weight of the true
 * b_i subject to every clause of phi; canonical optimum per R2/R3.
 * Algorithm: device packing (support restriction, dedup, subsumption,
 * ascending clause size), then ascending cardinality levels k = 1..k_max with
 * k_max = min(|support(phi+)|, |phi+ after subsumption|) (reading R13); each
 * level is enumerated in colex order by the persistent enumeration kernel;
 * unit weights stop at the first level with a witness, weights stop once the
 * k smallest weights sum to >= the incumbent. */
int gr_solve_pms(const gr_batch *in, gr_result *out, void *ws, size_t ws_bytes, gr_stream_t s);

/* (b) Exact MHS of phi+ (PAPER.md:11): cardinality only (w ignored, R10);
 * status GR_SAT_NEG_VIOLATED flags that the canonical MHS breaks phi-. */
int gr_mhs_exact(const gr_batch *in, gr_result *out, void *ws, size_t ws_bytes, gr_stream_t s);

/* (a) + (b) of one batch at once.  Unit weights (w == NULL, no k_start): one
 * enumeration decides both -- the MHS is phi+'s part of the PMS clause test --
 * on s_pms, and s_mhs waits for it.  Otherwise the PMS and MHS level loops
 * run interleaved on the two streams.  ws_bytes >= 2 * gr_workspace_bytes(in,
 * 0) (+256).  Results (status, assignment, cost, decided) are identical to
 * gr_solve_pms / gr_mhs_exact. */
int gr_solve_pms_mhs(const gr_batch *in, gr_result *out_pms, gr_result *out_mhs, void *ws,
                     size_t ws_bytes, gr_stream_t s_pms, gr_stream_t s_mhs);

/* (c) Greedy mhs of phi+ (Johnson 1974): repeatedly take the
 * variable hitting the most uncovered positive clauses (lowest index on ties,
 * R11), then reverse-delete in reverse pick order to a minimal hitting set
 * (R12); GR_SAT_NEG_VIOLATED if the set contains some N of phi- (PAPER.md:26).
 * One warp per instance; m <= 128 (W <= 2); duplicates are counted as given (R9).
 * cost = |S| (with GR_FLAG_WEIGHTED_GREEDY: the weighted greedy, cost = weight);
 * decided is not written. */
int gr_mhs_greedy(const gr_batch *in, gr_result *out, void *ws, size_t ws_bytes, gr_stream_t s);

/* ---- the composite Solve (Alg. 1 line `solve`) -------------
 * strategy GR_STRATEGY_MAXSAT: the (weighted) partial-MaxSAT optimum
 *   (= gr_solve_pms).
 * strategy GR_STRATEGY_MHS (the paper's default): the greedy mhs of phi+
 *   (= gr_mhs_greedy); every instance whose greedy set breaks phi- falls back
 *   to the MaxSAT solver and gets the gr_solve_pms result.
 *   With weights, a greedy answer's cost is its weight.
 * fell_back (device [B] int32, may be NULL): 1 where the fallback ran.
 * decided is 0 for instances answered by the greedy.  Workspace:
 * gr_workspace_bytes(in, 0). */
/* strategy GR_STRATEGY_MHS_FINAL: the mhs strategy's final query -- "a single
 *   query to a MaxSAT solver is needed to ensure that the number of b_i's
 *   being set to true is the minimum": the greedy mhs answer is
 *   computed, then every instance gets the (weighted) partial-MaxSAT optimum
 *   (= gr_solve_pms, decided counts included); fell_back[b] = 1 where that
 *   query changed the answer (the greedy set broke phi-, or the optimum is
 *   cheaper than the greedy set), 0 where the greedy answer was already
 *   minimum. */
enum { GR_STRATEGY_MHS = 0, GR_STRATEGY_MAXSAT = 1, GR_STRATEGY_MHS_FINAL = 2 };
int gr_solve(const gr_batch *in, int strategy, gr_result *out, int32_t *fell_back, void *ws,
             size_t ws_bytes, gr_stream_t s);

/* ---- sharded exact solving (the multi-GPU driver owns the collective) ----
 * gr_solve_pms / gr_mhs_exact are exactly:
 *     gr_exact_prepare(in, which, out, ..., &n);
 *     for (k = 1; n > 0; k++) { gr_exact_level(in, which, k, 0, 1, ...);
 *                               gr_exact_finish(in, which, k, out, ..., &n); }
 * With G GPUs, rank r calls gr_exact_level(in, k, r, G, ...), then all-reduces
 * (MIN, int64) the B level keys at gr_exact_level_keys(ws) before
 * gr_exact_finish -- every rank then holds the same state.  Level k's colex
 * rank range is cut into fixed chunks; shard r enumerates chunks c with
 * c % G == r.  which: 0 = PMS/WPMS, 1 = MHS. */
/* packs the batch, writes the results of trivially decided instances and
 * plans level 1; *n_active (host, may be NULL; if given the call synchronises
 * s) = instances that still search. */
int gr_exact_prepare(const gr_batch *in, int which, gr_result *out, void *ws, size_t ws_bytes,
                     gr_stream_t s, int32_t *n_active);
int gr_exact_level(const gr_batch *in, int which, int k, int shard, int nshard, void *ws,
                   size_t ws_bytes, gr_stream_t s);
int64_t *gr_exact_level_keys(const gr_batch *in, int which, void *ws);
/* commits level k, writes results of instances that finished, plans level
 * k+1 (chunk size adapted to the level's candidate count); *n_active (host)
 * = instances still searching.  Synchronises s only when n_active != NULL;
 * levels enumerated after every instance finished are no-ops, so a driver may
 * queue several levels per read-back (gr_solve_pms queues 4). */
int gr_exact_finish(const gr_batch *in, int which, int k, gr_result *out, void *ws,
                    size_t ws_bytes, gr_stream_t s, int32_t *n_active);

/* ---- fused PMS + MHS, step-wise (rank-range sharding of the fused walk) --
 * The pair session: gr_solve_pms_mhs's fused walk (unit weights, no k_start)
 * with the level loop owned by the caller, exactly like the gr_exact_*
 * session above -- ws holds two halves of gr_workspace_bytes(in, 0) (the PMS
 * state, then the MHS state).  Per level every rank calls
 * gr_pair_level(in, k, r, G, ...), all-reduces (MIN, int64) BOTH key arrays
 * (gr_pair_level_keys(in, ws, 0) -- PMS -- and (.., 1) -- MHS), then
 * gr_pair_finish.  Results equal gr_solve_pms / gr_mhs_exact.  Errors:
 * GR_EINVAL also for weights or k_start (the fused walk is cardinality-only). */
int gr_pair_prepare(const gr_batch *in, gr_result *out_pms, gr_result *out_mhs, void *ws,
                    size_t ws_bytes, gr_stream_t s, int32_t *n_active);
int gr_pair_level(const gr_batch *in, int k, int shard, int nshard, void *ws, size_t ws_bytes,
                  gr_stream_t s);
int64_t *gr_pair_level_keys(const gr_batch *in, void *ws, int which);
int gr_pair_finish(const gr_batch *in, int k, gr_result *out_pms, gr_result *out_mhs, void *ws,
                   size_t ws_bytes, gr_stream_t s, int32_t *n_active);

/* ---- greedy at scale: one phi+ as a variable-major bit matrix ----------- */
typedef struct {
  int32_t m;              /* host: number of variables (rows), >= 1 */
  int64_t n_pos;          /* host: number of positive clauses (columns), >= 0 */
  int64_t ld;             /* host: row stride in uint64 words, >= ceil(n_pos/64), multiple of 64 */
  const uint64_t *bits;   /* [m][ld] R[v][c/64] bit c%64 <=> b_{v+1} occurs in clause c;
                             bits at columns >= n_pos must be 0 */
  int32_t n_neg;          /* host: number of negative clauses */
  const uint64_t *neg;    /* [n_neg][ceil(m/64)] negative clause masks (may be NULL if n_neg == 0) */
  /* optional clause-major view of the same phi+ (the CSR given to
   * gr_pack_varmajor): with it the greedy keeps exact counts incrementally
   * (one 2 MiB row + the newly covered clauses' lists per pick, SURVEY
   * §8(f) f3) instead of re-streaming the matrix each pick; picks identical.
   * A clause must not list a variable twice.  NULL = recounting passes. */
  const int64_t *pos_off; /* [n_pos+1] or NULL */
  const void *pos_var;    /* [pos_off[n_pos]] int16 / int32 variable ids, or NULL */
  int32_t var_bytes;      /* 2 or 4 when pos_var is given; m <= 50000 (shared histogram) */
  const uint32_t *w;      /* [m] weights >= 1 or NULL: the weighted mhs (SURVEY §8(f) f4,
                             reading R20) -- pick the variable maximising uncovered hits /
                             weight, exact cross-multiplied comparison, lowest index on ties */
} gr_bitmatrix;

/* Row stride (words) the library uses for n_pos clauses: a multiple of 64. */
int64_t gr_bitmatrix_ld(int64_t n_pos);

/* Pack CSR variable lists into the variable-major bit matrix (clause packing
 * step a1).  off [n+1] int64, var [off[n]] int16 (var_bytes = 2) or int32
 * (var_bytes = 4), 0-based variable ids.  Every word of bits [m][ld] is
 * written (shared-memory tiles; ld a multiple of 16, as gr_bitmatrix_ld
 * gives), so it need not be cleared.  *d_bad (device int32, may be NULL) gets bit 1 if some id is outside
 * [0, m), bit 2 if some clause is empty (phi is then UNSAT, R6), bit 4 if a
 * clause lists a variable twice. */
int gr_pack_varmajor(int32_t m, int64_t n, const int64_t *off, const void *var, int var_bytes,
                     uint64_t *bits, int64_t ld, int32_t *d_bad, gr_stream_t s);
/* Same, clause-major [n][ceil(m/64)] masks (for phi-); out must be zeroed. */
int gr_pack_clausemajor(int32_t m, int64_t n, const int64_t *off, const void *var, int var_bytes,
                        uint64_t *masks, int32_t *d_bad, gr_stream_t s);

size_t gr_greedy_matrix_workspace_bytes(const gr_bitmatrix *in);

/* Greedy mhs over the bit matrix.  assign [ceil(m/64)] words (device);
 * status (device int32); picks (device, [m], or NULL): pick order before
 * pruning, padded with -1; n_picks (host, may be NULL) = number of picks.
 * Empty positive clauses must be reported by the caller (gr_pack_* d_bad). */
int gr_mhs_greedy_matrix(const gr_bitmatrix *in, uint64_t *assign, int32_t *status,
                         int32_t *picks, int32_t *n_picks, void *ws, size_t ws_bytes,
                         gr_stream_t s);

/* Shard hook for the multi-GPU greedy: counts[v] (device, [m] uint32) =
 * number of clauses c of this shard with U[c] = 1 and v in c. */
int gr_greedy_count_shard(const gr_bitmatrix *shard, const uint64_t *d_U, uint32_t *d_counts,
                          gr_stream_t s);

/* ---- greedy at scale from clause lists alone --------
 * The same greedy as gr_mhs_greedy_matrix (identical picks, pruned set and
 * phi- verdict) for one phi+ given only as clause -> variable lists, without
 * the variable-major bit matrix: the variable -> clause lists are built on
 * the device by a counting sort (~4 bytes per literal of workspace), every
 * pick walks its own list, covers the clauses still uncovered and decrements
 * the counts of their variables (exact counts, so the textbook argmax), all
 * picks in one cooperative launch; the reverse-delete keeps exact hit counts
 * per clause.  Ids outside [0, m): status GR_BADINPUT; an empty positive
 * clause: GR_UNSAT (R6).  Errors: GR_ETOOBIG for m > 51200 (shared-memory
 * histograms) or nnz / n_pos >= 2^32. */
typedef struct {
  int32_t m;              /* host: number of variables, >= 1 */
  int64_t n_pos;          /* host: number of positive clauses */
  int64_t nnz;            /* host: pos_off[n_pos], the number of literals */
  const int64_t *pos_off; /* [n_pos+1] device */
  const void *pos_var;    /* [nnz] device int16 / int32 variable ids (0-based); a clause
                             must not list a variable twice.  16-byte aligned (read in
                             16-byte groups, up to the next 16-byte boundary past nnz;
                             GR_EINVAL otherwise) */
  int32_t var_bytes;      /* 2 or 4 */
  int32_t n_neg;          /* host: number of negative clauses */
  const uint64_t *neg;    /* [n_neg][ceil(m/64)] device masks (gr_pack_clausemajor), or NULL */
  const uint32_t *w;      /* [m] weights >= 1 or NULL (the weighted mhs, R20) */
} gr_clauselists;
size_t gr_greedy_lists_workspace_bytes(const gr_clauselists *in);
/* assign [ceil(m/64)] words and status (device); picks (device [m] or NULL):
 * pick order before pruning, padded with -1; n_picks (host, may be NULL).
 * Synchronises s. */
int gr_mhs_greedy_lists(const gr_clauselists *in, uint64_t *assign, int32_t *status,
                        int32_t *picks, int32_t *n_picks, void *ws, size_t ws_bytes,
                        gr_stream_t s);

/* ---- column-sharded greedy (PAPER.md:24 greedy mhs) ---
 * Each rank owns a contiguous range of phi+'s clause columns as its own
 * gr_bitmatrix (same m, its own n_pos / ld / bits and, optionally, the CSR of
 * its clauses; phi- replicated).  The greedy's counts are sums over clauses,
 * so the caller all-reduces (SUM) the per-rank counts between steps and every
 * rank takes the same pick (ratio rule with weights, lowest index on ties,
 * readings R11/R20) -- picks identical to gr_mhs_greedy_matrix over the
 * whole matrix.  Protocol, all on stream s, one workspace per shard
 * (gr_greedy_shard_workspace_bytes, caller-owned device memory):
 *
 *   gr_greedy_shard_begin(sh, counts)        counts := this shard's counts
 *   repeat: all_reduce_sum(counts); gr_greedy_shard_step(sh, counts)
 *           (counts in: global counts; out: this shard's counts after the
 *            pick; a step after the last pick is a no-op)
 *   gr_greedy_shard_state(...)               n_picks, done (synchronises s)
 *   prune (reverse-delete, R12):
 *     gr_greedy_shard_private(sh, -1, flags) flags[j] |= pick j is the sole
 *                                            hitter of a clause of this shard
 *     all_reduce_max(flags); for j = n_picks-1 .. 0 with flags[j] == 0:
 *       flags[j] := 0; gr_greedy_shard_private(sh, j, flags);
 *       all_reduce_max(flags[j]); if still 0: removed[j] := 1 and
 *       gr_greedy_shard_remove(sh, j)
 *   gr_greedy_shard_finalize(sh, removed, assign, status)
 *
 * counts: device uint32 [m].  flags, removed: device int32 [m].  assign:
 * device [ceil(m/64)] words; status: device int32 (GR_SAT or
 * GR_SAT_NEG_VIOLATED).  Errors: GR_EINVAL (null pointer, bad matrix, j out
 * of range), GR_EWORKSPACE (workspace too small). */
size_t gr_greedy_shard_workspace_bytes(const gr_bitmatrix *shard);
int gr_greedy_shard_begin(const gr_bitmatrix *shard, uint32_t *d_counts, void *ws,
                          size_t ws_bytes, gr_stream_t s);
int gr_greedy_shard_step(const gr_bitmatrix *shard, uint32_t *d_counts, void *ws, size_t ws_bytes,
                         gr_stream_t s);
/* n_picks, done: host int32 (may be NULL); d_picks: device int32 [m] (may be
 * NULL) receives the pick order padded with -1. */
int gr_greedy_shard_state(const gr_bitmatrix *shard, const void *ws, size_t ws_bytes,
                          int32_t *n_picks, int32_t *done, int32_t *d_picks, gr_stream_t s);
int gr_greedy_shard_private(const gr_bitmatrix *shard, int32_t only, int32_t *d_flags, void *ws,
                            size_t ws_bytes, gr_stream_t s);
int gr_greedy_shard_remove(const gr_bitmatrix *shard, int32_t j, void *ws, size_t ws_bytes,
                           gr_stream_t s);
int gr_greedy_shard_finalize(const gr_bitmatrix *shard, const int32_t *d_removed,
                             uint64_t *assign, int32_t *status, void *ws, size_t ws_bytes,
                             gr_stream_t s);

/* ---- launch accounting and profiling ------------------------------------
 * Every kernel launch of the library is counted (gr_launch_count).  With
 * gr_profile(1) each launch is bracketed by CUDA events recorded on the
 * stream it is launched on; gr_profile(2) additionally runs the enumeration
 * kernel's work-counting instantiation (slower; for the roofline numerator).
 * gr_profile(mode) resets the statistics; gr_profile_read synchronises the
 * recorded events and returns one entry per kernel name. */
typedef struct {
  char name[48];
  int64_t launches;
  double ms;          /* summed event-timed duration of the launches */
  uint64_t work[8];   /* enum_kernel / queue_kernel in mode 2 (the roofline's units,
                         DESIGN.md §5): [0] positive clause tests, [1] negative clause
                         tests, [2] clauses read by subtree-refutation scans, [3] sub-blocks
                         tested, [4] candidates in tested sub-blocks, [5] lane windows
                         positioned, [6] tests + scans on 64-bit masks, [7] 0 */
} gr_kernel_stat;
int gr_profile(int mode);
int gr_profile_read(gr_kernel_stat *out, int max_stats);
unsigned long long gr_launch_count(void);

/* thread-local description of the last negative return */
const char *gr_last_error(void);
/* build identification, e.g. "grsolve 0.1 sm_100a" */
const char *gr_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GR_H */
