/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the Solve step of
 * GPURepair (arXiv 2011.08373).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path may link, load or
 * call this file: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it.  It shares no code, header,
 * table or constant with paper_2011_08373_b200/csrc (the CUDA path).
 *
 * What it computes (PAPER.md line numbers, LaTeX labels in parentheses):
 *   - clauses, phi+ / phi-            PAPER.md:5   (Se:preliminaries)
 *   - hitting set, mhs, MHS
 *   - PMS / WPMS
 *   - MaxSAT strategy: hard = phi, soft = {not b_1 .. not b_m}
 *                                     PAPER.md:24  (Se:repair_algorithm)
 *   - mhs strategy: Johnson's greedy  PAPER.md:24 (johnson1974approximation)
 *   - fallback when mhs breaks phi-   PAPER.md:26
 * and the readings of DESIGN.md §3 (R1..R12) where the paper is silent:
 *   R1 b_i <-> bit (i-1); R2 canonical optimum = smallest colex rank =
 *   numerically smallest mask; R3 weighted key (W, k, mask); R4 weights are
 *   integers >= 1, 0 => bad input; R6 empty clause => UNSAT; R8 bits >= m =>
 *   bad input; R11 greedy ties -> lowest index; R12 reverse-delete pruning in
 *   reverse pick order; R13 support restriction + k_max (optional `reduce`).
 *
 * All arithmetic is integer.  Parallelism (OpenMP) is only ever over
 * independent instances or over disjoint clause ranges whose partial counts
 * are summed -- never a reordering of the method's own steps.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* result codes (the oracle's own; the test maps them by meaning) */
enum { OR_SAT = 0, OR_UNSAT = 1, OR_SAT_NEG_VIOLATED = 2, OR_BADINPUT = 3 };
/* call-level errors */
enum { OR_OK = 0, OR_EINVAL = -1, OR_ETOOBIG = -2, OR_ENOMEM = -4 };

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void or_set_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}

static int popc64(uint64_t x) {
  int c = 0;
  while (x) { x &= x - 1; c++; }
  return c;
}

/* binomial coefficient C(n, k), n <= 64, by the product formula
 * C(n,k) = prod_{i=1..k} (n-k+i)/i (each partial product is an integer) */
static uint64_t binom(int n, int k) {
  if (k < 0 || k > n) return 0;
  unsigned __int128 r = 1;
  for (int i = 1; i <= k; i++) r = r * (unsigned)(n - k + i) / (unsigned)i;
  return (uint64_t)r;
}

/* a positive monotone clause P is satisfied by the assignment x
 * (bit i-1 set <=> b_i true) iff some b_i in P is true; a negative monotone
 * clause N is satisfied iff some b_i in N is false. */
static int clause_pos_sat(uint64_t x, uint64_t P) { return (x & P) != 0; }
static int clause_neg_sat(uint64_t x, uint64_t N) { return (x & N) != N; }

static int feasible(uint64_t x, const uint64_t *pos, int np, const uint64_t *neg, int nn) {
  for (int j = 0; j < np; j++) if (!clause_pos_sat(x, pos[j])) return 0;
  for (int j = 0; j < nn; j++) if (!clause_neg_sat(x, neg[j])) return 0;
  return 1;
}

/* WPMS objective: maximise the satisfied soft weight; the soft
 * clause (not b_i) is satisfied iff b_i is false, so this is the same as
 * minimising the weight of the true b_i (reading R5). */
static uint64_t cost_of(uint64_t x, const uint32_t *w) {
  uint64_t c = 0;
  for (int i = 0; i < 64; i++)
    if ((x >> i) & 1) c += w ? (uint64_t)w[i] : 1u;
  return c;
}

/* order-preserving relabel onto the support (pext) and back (pdep) */
static uint64_t compress(uint64_t x, uint64_t sup) {
  uint64_t r = 0; int j = 0;
  for (int i = 0; i < 64; i++)
    if ((sup >> i) & 1) { if ((x >> i) & 1) r |= 1ull << j; j++; }
  return r;
}
static uint64_t expand(uint64_t x, uint64_t sup) {
  uint64_t r = 0; int j = 0;
  for (int i = 0; i < 64; i++)
    if ((sup >> i) & 1) { if ((x >> j) & 1) r |= 1ull << i; j++; }
  return r;
}

/* Validation (readings R8, R4, R6).  bad_input: some bit >= m is set
 * (R8) or some weight of b_1..b_m is 0 (R4).  has_empty: some clause has no
 * literal -- an empty disjunction is false, so phi is UNSAT (R6). */
static int bad_input(int m, int W, int n, const uint64_t *masks, const uint32_t *w) {
  for (int j = 0; j < n; j++)
    for (int t = 0; t < W; t++) {
      uint64_t word = masks[(size_t)j * W + t];
      int lo = 64 * t;
      uint64_t allowed;
      if (m <= lo) allowed = 0;
      else if (m - lo >= 64) allowed = ~0ull;
      else allowed = (1ull << (m - lo)) - 1;
      if (word & ~allowed) return 1;
    }
  if (w) for (int i = 0; i < m; i++) if (w[i] == 0) return 1;
  return 0;
}
static int has_empty(int W, int n, const uint64_t *masks) {
  for (int j = 0; j < n; j++) {
    int empty = 1;
    for (int t = 0; t < W; t++) if (masks[(size_t)j * W + t]) empty = 0;
    if (empty) return 1;
  }
  return 0;
}
/* -1 if OK to proceed, else the status to report */
static int validate(int m, int W, int n, const uint64_t *masks, const uint32_t *w) {
  if (bad_input(m, W, n, masks, w)) return OR_BADINPUT;
  if (has_empty(W, n, masks)) return OR_UNSAT;
  return -1;
}

/*
 * Exact PMS / WPMS (MaxSAT strategy; definition).
 *   m <= 64, masks: (n_pos + n_neg) clauses x W words, positives first.
 *   w: NULL = unit weights (PMS), else w[0..m-1] >= 1 (WPMS).
 *   reduce = 0: enumerate all m variables, levels k = 0..m (the plain
 *              definition); reduce = 1: reading R13 -- restrict to the
 *              support of phi+ (order-preserving relabel), drop negative
 *              clauses touching non-support variables, stop at
 *              k_max = min(|support|, #clauses of phi+ not subsumed by
 *              another, equal clauses counted once).
 * Algorithm (levelled Gosper):
 *   for k = 0, 1, ...: (weighted: stop once S_k >= W_best, S_k = sum of the
 *   k smallest weights, reading R3)
 *     for x over all k-subsets in increasing numeric (= colex) order:
 *       if feasible(x): unit -> return x (smallest colex rank at the first
 *       feasible level, reading R2); weighted -> keep min (W(x), x).
 *     weighted: a level's best replaces the incumbent only if its W is
 *     strictly smaller (key (W, k, mask), reading R3).
 * Outputs: assign (1 word, 0 if UNSAT), cost (UINT64_MAX if UNSAT), status,
 *   decided = number of candidate subsets whose feasibility was tested.
 */
static int or_pms_from(int m, int W, int n_pos, int n_neg, const uint64_t *masks,
                       const uint32_t *w, int reduce, int kstart, uint64_t *assign,
                       uint64_t *cost, int32_t *status, uint64_t *decided);

int or_pms(int m, int W, int n_pos, int n_neg, const uint64_t *masks, const uint32_t *w,
           int reduce, uint64_t *assign, uint64_t *cost, int32_t *status, uint64_t *decided) {
  return or_pms_from(m, W, n_pos, n_neg, masks, w, reduce, 0, assign, cost, status, decided);
}

/* Incremental Solve: unit weights, levels below kstart are
 * not enumerated (the caller knows they hold no feasible set). */
int or_pms_kstart(int m, int W, int n_pos, int n_neg, const uint64_t *masks, int reduce, int kstart,
                  uint64_t *assign, uint64_t *cost, int32_t *status, uint64_t *decided) {
  return or_pms_from(m, W, n_pos, n_neg, masks, NULL, reduce, kstart, assign, cost, status, decided);
}

static int or_pms_from(int m, int W, int n_pos, int n_neg, const uint64_t *masks,
                       const uint32_t *w, int reduce, int kstart, uint64_t *assign,
                       uint64_t *cost, int32_t *status, uint64_t *decided) {
  if (m < 0 || W < 1 || W > 2 || n_pos < 0 || n_neg < 0) return OR_EINVAL;
  for (int t = 0; t < W; t++) assign[t] = 0;
  *cost = UINT64_MAX; *decided = 0;
  int n = n_pos + n_neg;
  int v = validate(m, W, n, masks, w);
  if (v >= 0) { *status = v; return OR_OK; }
  if (!reduce && m > 64) return OR_ETOOBIG;
  uint64_t *pos = (uint64_t *)malloc(sizeof(uint64_t) * (n_pos + 1));
  uint64_t *neg = (uint64_t *)malloc(sizeof(uint64_t) * (n_neg + 1));
  uint32_t wr[64];
  if (!pos || !neg) { free(pos); free(neg); return OR_ENOMEM; }
  /* sup[t]: the enumerated variables (word t) */
  uint64_t sup[2] = {0, 0};
  int np = n_pos, nn = 0, me = m, kmax = m;
  if (reduce) {
    for (int j = 0; j < n_pos; j++) for (int t = 0; t < W; t++) sup[t] |= masks[(size_t)j * W + t];
    me = popc64(sup[0]) + popc64(sup[1]);
    if (me > 64) { free(pos); free(neg); return OR_ETOOBIG; }
    for (int j = 0; j < n_pos; j++)
      pos[j] = compress(masks[(size_t)j * W], sup[0]) |
               (W > 1 ? compress(masks[(size_t)j * W + 1], sup[1]) << popc64(sup[0]) : 0);
    for (int j = 0; j < n_neg; j++) {
      const uint64_t *N = masks + (size_t)(n_pos + j) * W;
      int inside = 1;
      for (int t = 0; t < W; t++) if (N[t] & ~sup[t]) inside = 0;
      if (inside)
        neg[nn++] = compress(N[0], sup[0]) | (W > 1 ? compress(N[1], sup[1]) << popc64(sup[0]) : 0);
    }
    /* k_max (reading R13): a minimal hitting set has at most one element per
     * clause of phi+ that no other clause subsumes (a private clause of x
     * can be taken inside every clause it contains, and equal clauses count
     * once), and an optimum is a minimal hitting set (dropping a variable
     * keeps phi- satisfied and lowers the weight) */
    int nmin = 0;
    for (int j = 0; j < n_pos; j++) {
      int subsumed = 0;
      for (int i = 0; i < n_pos && !subsumed; i++)
        if (i != j && (pos[i] & ~pos[j]) == 0 && (pos[i] != pos[j] || i < j)) subsumed = 1;
      nmin += !subsumed;
    }
    kmax = me < nmin ? me : nmin;
  } else {
    sup[0] = (m == 64) ? ~0ull : ((1ull << m) - 1);
    for (int j = 0; j < n_pos; j++) pos[j] = masks[(size_t)j * W];
    for (int j = 0; j < n_neg; j++) neg[nn++] = masks[(size_t)(n_pos + j) * W];
  }
  { int j = 0;
    for (int t = 0; t < 2; t++) for (int i = 0; i < 64; i++) if ((sup[t] >> i) & 1) wr[j++] = w ? w[64 * t + i] : 1u; }
  /* sorted weights for S_k (insertion sort, me <= 64) */
  uint32_t ws[64];
  for (int i = 0; i < me; i++) ws[i] = wr[i];
  for (int i = 1; i < me; i++) { uint32_t t = ws[i]; int j = i - 1; while (j >= 0 && ws[j] > t) { ws[j + 1] = ws[j]; j--; } ws[j + 1] = t; }

  int found = 0; uint64_t best_x = 0, best_W = UINT64_MAX, Sk = 0, nd = 0;
  for (int k = 0; k <= kmax; k++) {
    if (k > 0) Sk += ws[k - 1];
    if (w && found && Sk >= best_W) break;
    if (!w && k > 0 && k < kstart) continue;  /* level 0 is always tested */
    uint64_t cnt = binom(me, k);
    uint64_t x = (k == 64) ? ~0ull : ((1ull << k) - 1);
    int lvl_found = 0; uint64_t lvl_x = 0, lvl_W = UINT64_MAX;
    for (uint64_t i = 0; i < cnt; i++) {
      nd++;
      if (feasible(x, pos, np, neg, nn)) {
        if (!w) { lvl_found = 1; lvl_x = x; lvl_W = (uint64_t)k; break; }
        uint64_t c = cost_of(x, wr);
        if (!lvl_found || c < lvl_W) { lvl_found = 1; lvl_x = x; lvl_W = c; }
      }
      if (i + 1 < cnt) { /* Gosper's hack (HAKMEM 175): next k-subset in numeric order */
        uint64_t c = x & (~x + 1), r = x + c;
        x = (((r ^ x) >> 2) / c) | r;
      }
    }
    if (lvl_found && (!found || lvl_W < best_W)) { found = 1; best_x = lvl_x; best_W = lvl_W; }
    if (!w && found) break;
  }
  *decided = nd;
  if (found) {
    if (reduce) {
      assign[0] = expand(best_x, sup[0]);
      if (W > 1) assign[1] = expand(best_x >> popc64(sup[0]), sup[1]);
    } else {
      assign[0] = best_x;
    }
    *cost = cost_of(assign[0], w) + (W > 1 ? cost_of(assign[1], w ? w + 64 : NULL) : 0);
    *status = OR_SAT;
  } else {
    *status = OR_UNSAT;
  }
  free(pos); free(neg);
  return OR_OK;
}

/* Independent second oracle for m <= 30: scan ALL 2^m assignments and take
 * the minimum of the key (W(x), popcount(x), x) over feasible x. */
int or_pms_brute(int m, int W, int n_pos, int n_neg, const uint64_t *masks, const uint32_t *w,
                 uint64_t *assign, uint64_t *cost, int32_t *status) {
  *assign = 0; *cost = UINT64_MAX;
  int v = validate(m, W, n_pos + n_neg, masks, w);
  if (v >= 0) { *status = v; return OR_OK; }
  if (m > 30) return OR_ETOOBIG;
  const uint64_t *pos = NULL; uint64_t *p = malloc(sizeof(uint64_t) * (n_pos + n_neg + 1));
  for (int j = 0; j < n_pos + n_neg; j++) p[j] = masks[(size_t)j * W];
  pos = p;
  int found = 0; uint64_t bx = 0, bW = 0; int bk = 0;
  for (uint64_t x = 0; x < (1ull << m); x++) {
    if (!feasible(x, pos, n_pos, pos + n_pos, n_neg)) continue;
    uint64_t c = cost_of(x, w); int k = popc64(x);
    if (!found || c < bW || (c == bW && (k < bk || (k == bk && x < bx)))) { found = 1; bx = x; bW = c; bk = k; }
  }
  free(p);
  if (found) { *assign = bx; *cost = bW; *status = OR_SAT; } else *status = OR_UNSAT;
  return OR_OK;
}

/* Exact MHS over phi+ (no smaller hitting set exists; reading
 * R10: cardinality only, weights ignored), canonical = smallest colex rank.
 * The status additionally flags phi-: SAT_NEG_VIOLATED iff some negative
 * clause N has all its b_i true in the MHS (N subset of S). */
int or_mhs(int m, int W, int n_pos, int n_neg, const uint64_t *masks, int reduce,
           uint64_t *assign, uint64_t *cost, int32_t *status, uint64_t *decided) {
  for (int t = 0; t < W; t++) assign[t] = 0;
  *cost = UINT64_MAX; *decided = 0;
  if (bad_input(m, W, n_pos + n_neg, masks, NULL)) { *status = OR_BADINPUT; return OR_OK; }
  if (has_empty(W, n_pos, masks)) { *status = OR_UNSAT; return OR_OK; }
  int rc = or_pms(m, W, n_pos, 0, masks, NULL, reduce, assign, cost, status, decided);
  if (rc != OR_OK || *status != OR_SAT) return rc;
  for (int j = 0; j < n_neg; j++) {
    const uint64_t *N = masks + (size_t)(n_pos + j) * W;
    int all_true = 1;
    for (int t = 0; t < W; t++) if ((assign[t] & N[t]) != N[t]) all_true = 0;
    if (all_true) { *status = OR_SAT_NEG_VIOLATED; break; }
  }
  return OR_OK;
}

/*
 * Greedy minimal hitting set over phi+ (mhs strategy; Johnson
 * 1974), textbook recount form, then reverse-delete (reading R12), then the
 * phi- check that triggers the MaxSAT fallback.
 *   clauses as variable lists (0-based ids), CSR: pos_off[n_pos+1], pos_var.
 *   U = all positive clauses; repeat while U non-empty:
 *     c[v] = |{P in U : v in P}| for every v;
 *     v* = the lowest v with c[v] = max c          (reading R11)
 *     S.append(v*); U = {P in U : v* not in P}
 *   for x in reversed(S) (weighted mhs: by descending weight, equal weights
 *   in reverse pick order -- reading R12): drop x if every P in phi+ meets
 *   S \ {x}.
 *   status = SAT_NEG_VIOLATED if some N in phi- has N subset of S, else SAT.
 * Outputs: picks[0..n_unpruned-1] = pick order (before pruning);
 *   in_S[m] = final (pruned) set as 0/1 bytes; n_final = |S| after pruning.
 * Counting over clause ranges is parallel (per-thread counts then summed).
 */
static int greedy_core(int m, int64_t n_pos, const int64_t *pos_off, const int32_t *pos_var,
                       int64_t n_neg, const int64_t *neg_off, const int32_t *neg_var,
                       const uint32_t *w, int32_t *picks, int32_t *n_unpruned, uint8_t *in_S,
                       int32_t *n_final, int32_t *status);

int or_greedy(int m, int64_t n_pos, const int64_t *pos_off, const int32_t *pos_var,
              int64_t n_neg, const int64_t *neg_off, const int32_t *neg_var,
              int32_t *picks, int32_t *n_unpruned, uint8_t *in_S, int32_t *n_final,
              int32_t *status) {
  return greedy_core(m, n_pos, pos_off, pos_var, n_neg, neg_off, neg_var, NULL, picks,
                     n_unpruned, in_S, n_final, status);
}

/* Weighted mhs ("weighted mhs"; SPEC.md:248 ratio rule, reading
 * R20): each step picks the v maximising c[v] / w[v] (the uncovered clauses
 * it hits per unit weight; Chvatal 1979), compared exactly as
 * c[a] * w[b] > c[b] * w[a], lowest index on ties; then the same
 * reverse-delete and phi- check. */
int or_greedy_w(int m, int64_t n_pos, const int64_t *pos_off, const int32_t *pos_var,
                int64_t n_neg, const int64_t *neg_off, const int32_t *neg_var, const uint32_t *w,
                int32_t *picks, int32_t *n_unpruned, uint8_t *in_S, int32_t *n_final,
                int32_t *status) {
  return greedy_core(m, n_pos, pos_off, pos_var, n_neg, neg_off, neg_var, w, picks, n_unpruned,
                     in_S, n_final, status);
}

static int greedy_core(int m, int64_t n_pos, const int64_t *pos_off, const int32_t *pos_var,
                       int64_t n_neg, const int64_t *neg_off, const int32_t *neg_var,
                       const uint32_t *w, int32_t *picks, int32_t *n_unpruned, uint8_t *in_S,
                       int32_t *n_final, int32_t *status) {
  *n_unpruned = 0; *n_final = 0;
  if (m < 0 || n_pos < 0 || n_neg < 0) return OR_EINVAL;
  memset(in_S, 0, (size_t)m);
  for (int64_t e = 0; e < pos_off[n_pos]; e++) if (pos_var[e] < 0 || pos_var[e] >= m) { *status = OR_BADINPUT; return OR_OK; }
  for (int64_t e = 0; e < neg_off[n_neg]; e++) if (neg_var[e] < 0 || neg_var[e] >= m) { *status = OR_BADINPUT; return OR_OK; }
  for (int64_t j = 0; j < n_pos; j++) if (pos_off[j + 1] == pos_off[j]) { *status = OR_UNSAT; return OR_OK; }
  uint8_t *covered = calloc((size_t)n_pos + 1, 1);
  int nt = or_num_threads();
  int64_t *cnt_all = calloc((size_t)nt * (m + 1), sizeof(int64_t));
  int64_t *cnt = calloc((size_t)m + 1, sizeof(int64_t));
  if (!covered || !cnt_all || !cnt) { free(covered); free(cnt_all); free(cnt); return OR_ENOMEM; }
  int nS = 0;
  for (;;) {
    memset(cnt_all, 0, sizeof(int64_t) * (size_t)nt * (m + 1));
#pragma omp parallel
    {
      int t = 0;
#ifdef _OPENMP
      t = omp_get_thread_num();
#endif
      int64_t *my = cnt_all + (size_t)t * (m + 1);
#pragma omp for schedule(static)
      for (int64_t j = 0; j < n_pos; j++) {
        if (covered[j]) continue;
        for (int64_t e = pos_off[j]; e < pos_off[j + 1]; e++) my[pos_var[e]]++;
      }
    }
    for (int v = 0; v < m; v++) { int64_t s = 0; for (int t = 0; t < nt; t++) s += cnt_all[(size_t)t * (m + 1) + v]; cnt[v] = s; }
    int best = -1;
    for (int v = 0; v < m; v++) {
      if (best < 0) { best = v; continue; }
      if (!w) { if (cnt[v] > cnt[best]) best = v; }
      else if ((unsigned __int128)cnt[v] * w[best] > (unsigned __int128)cnt[best] * w[v]) best = v;
    }
    if (best < 0 || cnt[best] == 0) break; /* U is empty */
    picks[nS++] = best;
    in_S[best] = 1;
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n_pos; j++) {
      if (covered[j]) continue;
      for (int64_t e = pos_off[j]; e < pos_off[j + 1]; e++) if (pos_var[e] == best) { covered[j] = 1; break; }
    }
  }
  *n_unpruned = nS;
  /* reverse-delete: x is dropped if every positive clause meets S \ {x}.
   * Order (reading R12): unit weights -- reverse pick order; weighted mhs --
   * descending weight ("in descending-weight order"), equal
   * weights in reverse pick order.  ord[] lists pick positions in that order
   * (insertion sort: stable, plain). */
  int *ord = malloc(sizeof(int) * ((size_t)nS + 1));
  if (!ord) { free(covered); free(cnt_all); free(cnt); return OR_ENOMEM; }
  for (int i = 0; i < nS; i++) {
    int p = nS - 1 - i, j = i - 1; /* reverse pick order first */
    while (w && j >= 0 && w[picks[ord[j]]] < w[picks[p]]) { ord[j + 1] = ord[j]; j--; }
    ord[j + 1] = p;
  }
  for (int r = 0; r < nS; r++) {
    int x = picks[ord[r]];
    in_S[x] = 0;
    int64_t unhit = 0;
#pragma omp parallel for schedule(static) reduction(+ : unhit)
    for (int64_t j = 0; j < n_pos; j++) {
      int hit = 0;
      for (int64_t e = pos_off[j]; e < pos_off[j + 1]; e++) if (in_S[pos_var[e]]) { hit = 1; break; }
      if (!hit) unhit++;
    }
    if (unhit) in_S[x] = 1;
  }
  free(ord);
  int nf = 0;
  for (int v = 0; v < m; v++) nf += in_S[v];
  *n_final = nf;
  *status = OR_SAT;
  for (int64_t j = 0; j < n_neg; j++) {
    int all_true = 1;
    for (int64_t e = neg_off[j]; e < neg_off[j + 1]; e++) if (!in_S[neg_var[e]]) { all_true = 0; break; }
    if (all_true) { *status = OR_SAT_NEG_VIOLATED; break; }
  }
  free(covered); free(cnt_all); free(cnt);
  return OR_OK;
}

/* greedy over mask-encoded clauses (W words each): unpack to variable lists
 * and run or_greedy.  assign: W words out. picks: capacity m. */
int or_greedy_masks_w(int m, int W, int n_pos, int n_neg, const uint64_t *masks,
                      const uint32_t *w, uint64_t *assign, int32_t *picks, int32_t *n_unpruned,
                      int32_t *status);
int or_greedy_masks(int m, int W, int n_pos, int n_neg, const uint64_t *masks,
                    uint64_t *assign, int32_t *picks, int32_t *n_unpruned, int32_t *status) {
  return or_greedy_masks_w(m, W, n_pos, n_neg, masks, NULL, assign, picks, n_unpruned, status);
}
int or_greedy_masks_w(int m, int W, int n_pos, int n_neg, const uint64_t *masks,
                      const uint32_t *w, uint64_t *assign, int32_t *picks, int32_t *n_unpruned,
                      int32_t *status) {
  int n = n_pos + n_neg;
  for (int t = 0; t < W; t++) assign[t] = 0;
  *n_unpruned = 0;
  if (bad_input(m, W, n, masks, w)) { *status = OR_BADINPUT; return OR_OK; }
  int64_t *off = malloc(sizeof(int64_t) * (n + 2));
  int32_t *var = malloc(sizeof(int32_t) * ((size_t)n * 64 * W + 1));
  uint8_t *inS = malloc((size_t)m + 1);
  if (!off || !var || !inS) { free(off); free(var); free(inS); return OR_ENOMEM; }
  off[0] = 0;
  for (int j = 0; j < n; j++) {
    int64_t e = off[j];
    for (int i = 0; i < 64 * W; i++) if ((masks[(size_t)j * W + i / 64] >> (i % 64)) & 1) var[e++] = i;
    off[j + 1] = e;
  }
  int32_t nf;
  int rc = greedy_core(m, n_pos, off, var, n_neg, off + n_pos, var, w, picks, n_unpruned, inS, &nf, status);
  if (rc == OR_OK && *status != OR_UNSAT && *status != OR_BADINPUT)
    for (int i = 0; i < m; i++) if (inS[i]) assign[i / 64] |= 1ull << (i % 64);
  free(off); free(var); free(inS);
  return rc;
}

/* The composite Solve: mhs strategy = greedy over phi+; if
 * the greedy set breaks phi- ("results in unsatisfiability"), fall back to
 * the MaxSAT solver (or_pms).  cost: weight (or size) of the returned set. */
int or_solve_mhs(int m, int W, int n_pos, int n_neg, const uint64_t *masks, const uint32_t *w,
                 int reduce, int weighted_greedy, uint64_t *assign, uint64_t *cost,
                 int32_t *status, uint64_t *decided, int32_t *fell_back) {
  int32_t *pk = malloc(sizeof(int32_t) * (m + 1)), nu;
  int rc = or_greedy_masks_w(m, W, n_pos, n_neg, masks, weighted_greedy ? w : NULL, assign, pk,
                             &nu, status);
  free(pk);
  *decided = 0;
  *fell_back = 0;
  if (rc != OR_OK) return rc;
  if (*status == OR_SAT_NEG_VIOLATED) {
    *fell_back = 1;
    return or_pms(m, W, n_pos, n_neg, masks, w, reduce, assign, cost, status, decided);
  }
  if (*status != OR_SAT) { *cost = UINT64_MAX; return OR_OK; }
  uint64_t c = 0;
  for (int t = 0; t < W; t++) c += cost_of(assign[t], w ? w + 64 * t : NULL);
  *cost = c;
  return OR_OK;
}

/* ---- batch drivers: independent instances in parallel ------------------ */
/* which: 0 = PMS/WPMS (w may be NULL), 1 = MHS (weights ignored), 2 = greedy,
 * 3 = composite Solve, mhs strategy with MaxSAT fallback (decided[b] = 1 where
 * the fallback ran, else 0 -- the fallback flag, not a candidate count),
 * 4 = weighted greedy (w), 5 = composite Solve with the weighted greedy */
int or_batch(int which, int B, int W, const int32_t *m, const int64_t *off, const int32_t *n_pos,
             const uint64_t *masks, const uint32_t *w, int wstride, int reduce,
             uint64_t *assign /*[B][W]*/, uint64_t *cost, int32_t *status, uint64_t *decided) {
  int err = OR_OK;
#pragma omp parallel for schedule(dynamic, 1)
  for (int b = 0; b < B; b++) {
    int n = (int)(off[b + 1] - off[b]);
    const uint64_t *mk = masks + (size_t)off[b] * W;
    int np = n_pos[b], nn = n - n_pos[b];
    uint64_t c = UINT64_MAX, d = 0; int32_t s = 0; int rc = OR_OK;
    uint64_t *a = assign + (size_t)b * W;
    for (int t = 0; t < W; t++) a[t] = 0;
    if (which == 0) rc = or_pms(m[b], W, np, nn, mk, w ? w + (size_t)b * wstride : NULL, reduce, a, &c, &s, &d);
    else if (which == 1) rc = or_mhs(m[b], W, np, nn, mk, reduce, a, &c, &s, &d);
    else if (which == 3 || which == 5) {
      int32_t fb = 0;
      rc = or_solve_mhs(m[b], W, np, nn, mk, w ? w + (size_t)b * wstride : NULL, reduce, which == 5,
                        a, &c, &s, &d, &fb);
      d = (uint64_t)fb;
    }
    else {
      const uint32_t *wb = (which == 4 && w) ? w + (size_t)b * wstride : NULL;
      int32_t *pk = malloc(sizeof(int32_t) * (m[b] + 1)); int32_t nu;
      rc = or_greedy_masks_w(m[b], W, np, nn, mk, wb, assign + (size_t)b * W, pk, &nu, &s);
      c = 0;
      for (int t = 0; t < W; t++) c += wb ? cost_of(assign[(size_t)b * W + t], wb + 64 * t)
                                         : (uint64_t)popc64(assign[(size_t)b * W + t]);
      if (s == OR_UNSAT || s == OR_BADINPUT) c = UINT64_MAX;
      free(pk);
    }
    cost[b] = c; status[b] = s; if (decided) decided[b] = d;
    if (rc == OR_ETOOBIG) { s = -1; rc = OR_OK; }  /* support > 64: no oracle value */
    status[b] = s;
    if (rc != OR_OK) {
#pragma omp critical
      err = rc;
    }
  }
  return err;
}

/* Minimum feasible mask over the product of disjoint groups (one variable per
 * group; gbits = single-bit masks, group g owns gbits[goff[g]..goff[g+1]-1]).
 * Used for pin P15: when phi+ contains G disjoint clauses and
 * a feasible G-set exists, every optimal set picks exactly one variable per
 * group, so the canonical optimum is the minimum feasible product element.
 * Returns the number of feasible product elements; *best = min mask. */
uint64_t or_min_feasible_product(int G, const int64_t *goff, const uint64_t *gbits,
                                 int n_pos, int n_neg, const uint64_t *masks, uint64_t *best) {
  uint64_t total = 1;
  for (int g = 0; g < G; g++) total *= (uint64_t)(goff[g + 1] - goff[g]);
  uint64_t nfeas = 0, bmin = UINT64_MAX;
#pragma omp parallel for schedule(static) reduction(+ : nfeas) reduction(min : bmin)
  for (uint64_t t = 0; t < total; t++) {
    uint64_t x = 0, r = t;
    for (int g = 0; g < G; g++) {
      uint64_t sz = (uint64_t)(goff[g + 1] - goff[g]);
      x |= gbits[goff[g] + (int64_t)(r % sz)];
      r /= sz;
    }
    if (feasible(x, masks, n_pos, masks + n_pos, n_neg)) { nfeas++; if (x < bmin) bmin = x; }
  }
  *best = bmin;
  return nfeas;
}

/* plain feasibility of one assignment (W = 1) -- used by property tests */
int or_feasible(uint64_t x, int n_pos, int n_neg, const uint64_t *masks) {
  return feasible(x, masks, n_pos, masks + n_pos, n_neg);
}
