// greedy_small.cu -- gr_mhs_greedy: Johnson's greedy mhs for a
// batch of small instances (m <= 128), one warp per instance.
//
//   U = phi+; repeat { c[v] = |{P in U : v in P}|; v* = lowest argmax (R11);
//   S += v*; U -= {P : v* in P} } until U is empty; reverse-delete in reverse
//   pick order (R12; weighted mhs: descending weight); status SAT_NEG_VIOLATED if some N in phi- is a subset
//   of S.
//
// Lane v (and v+32, v+64, v+96) owns the counter of variable v; the uncovered
// set U is a bitmap in shared memory whose 32-bit words are owned round-robin
// by the lanes when marking; argmax = warp max-reduction of the packed key
// (count << 8 | 255 - v).
//
// Weighted mhs (GR_FLAG_WEIGHTED_GREEDY): the
// pick maximises count[v] / w[v], compared exactly as c_a * w_b > c_b * w_a
// with the lowest index on ties (reading R20); warp reduction over
// (count, weight, v) triples.
#include "common.cuh"

namespace {
constexpr int MAXC = 4096;

__global__ void __launch_bounds__(32) greedy_small_kernel(gr_batch in, gr_result out) {
  extern __shared__ u64 sg[];  // [max_clauses][2] masks, then U bitmap words
  const int b = blockIdx.x, lane = threadIdx.x;
  u64 *C = sg;
  u32 *U = (u32 *)(sg + 2 * (size_t)in.max_clauses);
  __shared__ int s_picks[128], s_order[128];
  const int64_t lo = in.off[b], n64 = in.off[b + 1] - lo;
  const int m = in.m[b], np = in.n_pos[b], W = in.W;
  const bool wgt = (in.flags & GR_FLAG_WEIGHTED_GREEDY) && in.w;
  const uint32_t *wb = wgt ? in.w + (size_t)b * in.wstride : nullptr;
  int status = GR_SAT;
  u64 S0 = 0, S1 = 0;
  if (n64 < 0 || n64 > in.max_clauses || np < 0 || np > n64 || m < 0 || m > 64 * W) {
    status = GR_BADINPUT;
  } else {
    const int n = (int)n64;
    const u64 al0 = m >= 64 ? ~0ull : ((1ull << m) - 1);
    const u64 al1 = m >= 128 ? ~0ull : (m <= 64 ? 0ull : ((1ull << (m - 64)) - 1));
    int bad = 0, empty = 0;
    for (int j = lane; j < n; j += 32) {
      const u64 x0 = in.masks[(lo + j) * W], x1 = W > 1 ? in.masks[(lo + j) * W + 1] : 0;
      C[2 * j] = x0;
      C[2 * j + 1] = x1;
      bad |= ((x0 & ~al0) | (x1 & ~al1)) != 0;
      empty |= (j < np) && !(x0 | x1);
    }
    const int nw = (np + 31) / 32;
    for (int q = lane; q < nw; q += 32) {
      const int rem = np - 32 * q;
      U[q] = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
    }
    __syncwarp();
    if (wgt)
      for (int i = lane; i < m; i += 32) bad |= wb[i] == 0;  // R4
    bad = __any_sync(0xffffffffu, bad);
    empty = __any_sync(0xffffffffu, empty);
    if (bad) status = GR_BADINPUT;
    else if (empty) status = GR_UNSAT;  // no variable hits an empty clause (R6)
    else {
      int npk = 0;
      for (;;) {
        // counts of the lane's variables over the uncovered clauses
        int cnt[4] = {0, 0, 0, 0};
        for (int q = 0; q < nw; q++) {
          u32 u = U[q];
          while (u) {
            const int j = 32 * q + (__ffs(u) - 1);
            u &= u - 1;
            const u64 x0 = C[2 * j], x1 = C[2 * j + 1];
            cnt[0] += (int)((x0 >> lane) & 1);
            cnt[1] += (int)((x0 >> (lane + 32)) & 1);
            cnt[2] += (int)((x1 >> lane) & 1);
            cnt[3] += (int)((x1 >> (lane + 32)) & 1);
          }
        }
        int v = -1;
        if (!wgt) {
          u32 key = 0;
          for (int q = 0; q < 4; q++) {
            const int vq = lane + 32 * q;
            if (vq < m && cnt[q] > 0) {
              const u32 kq = ((u32)cnt[q] << 8) | (u32)(255 - vq);
              key = kq > key ? kq : key;
            }
          }
          for (int o = 16; o; o >>= 1) {
            const u32 o2 = __shfl_xor_sync(0xffffffffu, key, o);
            key = o2 > key ? o2 : key;
          }
          if (!key) break;  // U is empty
          v = 255 - (int)(key & 0xff);
        } else {
          // best (count, weight, index) of the lane, then of the warp
          u32 bc = 0, bw = 1;
          int bv = 0x7fffffff;
          for (int q = 0; q < 4; q++) {
            const int vq = lane + 32 * q;
            if (vq < m && cnt[q] > 0) {
              const u32 wq = wb[vq];
              const u64 l = (u64)cnt[q] * bw, r = (u64)bc * wq;
              if (l > r || (l == r && vq < bv)) { bc = (u32)cnt[q]; bw = wq; bv = vq; }
            }
          }
          for (int o = 16; o; o >>= 1) {
            const u32 oc = __shfl_xor_sync(0xffffffffu, bc, o);
            const u32 ow = __shfl_xor_sync(0xffffffffu, bw, o);
            const int ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const u64 l = (u64)oc * bw, r = (u64)bc * ow;
            if (l > r || (l == r && ov < bv)) { bc = oc; bw = ow; bv = ov; }
          }
          if (!bc) break;  // U is empty
          v = bv;
        }
        if (lane == 0) s_picks[npk] = v;
        npk++;
        if (v < 64) S0 |= 1ull << v; else S1 |= 1ull << (v - 64);
        // mark the clauses that contain v as covered
        for (int q = lane; q < nw; q += 32) {
          u32 u = U[q], nu = u;
          while (u) {
            const int bit = __ffs(u) - 1;
            u &= u - 1;
            const int j = 32 * q + bit;
            const u64 x = v < 64 ? C[2 * j] : C[2 * j + 1];
            if ((x >> (v & 63)) & 1) nu &= ~(1u << bit);
          }
          U[q] = nu;
        }
        __syncwarp();
      }
      // reverse-delete: drop x if every positive clause meets S \ {x}.
      // Order (R12): reverse pick order; weighted mhs: descending weight,
      // equal weights in reverse pick order -- position of
      // pick i = #{j : w_j > w_i or (w_j == w_i and j > i)}
      if (wgt) {
        __syncwarp();
        for (int i = lane; i < npk; i += 32) {
          const u32 wi = wb[s_picks[i]];
          int r = 0;
          for (int j = 0; j < npk; j++) {
            const u32 wj = wb[s_picks[j]];
            r += wj > wi || (wj == wi && j > i);
          }
          s_order[r] = s_picks[i];
        }
        __syncwarp();
      }
      for (int q = 0; q < npk; q++) {
        const int x = wgt ? s_order[q] : s_picks[npk - 1 - q];
        const u64 T0 = x < 64 ? (S0 & ~(1ull << x)) : S0;
        const u64 T1 = x >= 64 ? (S1 & ~(1ull << (x - 64))) : S1;
        int ok = 1;
        for (int j = lane; j < np; j += 32) ok &= ((C[2 * j] & T0) | (C[2 * j + 1] & T1)) != 0;
        if (__all_sync(0xffffffffu, ok)) { S0 = T0; S1 = T1; }
      }
      // phi- check
      int viol = 0;
      for (int j = np + lane; j < n; j += 32)
        viol |= ((C[2 * j] & ~S0) | (C[2 * j + 1] & ~S1)) == 0;
      if (__any_sync(0xffffffffu, viol)) status = GR_SAT_NEG_VIOLATED;
    }
  }
  if (lane == 0) {
    const bool ok = status == GR_SAT || status == GR_SAT_NEG_VIOLATED;
    out.assign[(size_t)b * W] = ok ? S0 : 0;
    if (W > 1) out.assign[(size_t)b * W + 1] = ok ? S1 : 0;
    u64 cost = (u64)(__popcll(S0) + __popcll(S1));
    if (wgt) {
      cost = 0;
      for (u64 a = S0; a; a &= a - 1) cost += wb[__ffsll((long long)a) - 1];
      for (u64 a = S1; a; a &= a - 1) cost += wb[64 + __ffsll((long long)a) - 1];
    }
    out.cost[b] = ok ? cost : ~0ull;
    out.status[b] = status;
  }
}
}  // namespace

extern "C" int gr_mhs_greedy(const gr_batch *in, gr_result *out, void *ws, size_t ws_bytes,
                             gr_stream_t s) {
  (void)ws;
  (void)ws_bytes;
  if (!in || !out || !out->assign || !out->cost || !out->status) { gr_set_error("null argument"); return GR_EINVAL; }
  if (in->B < 1 || (in->W != 1 && in->W != 2)) { gr_set_error("B < 1 or W not in {1,2}"); return GR_EINVAL; }
  if (!in->m || !in->off || !in->n_pos || (!in->masks && in->total_clauses > 0)) { gr_set_error("null device pointer"); return GR_EINVAL; }
  if (in->max_clauses < 0) { gr_set_error("max_clauses < 0"); return GR_EINVAL; }
  if (in->max_clauses > MAXC) { gr_set_error("max_clauses > 4096 for gr_mhs_greedy"); return GR_ETOOBIG; }
  const size_t smem = (size_t)in->max_clauses * 16 + ((size_t)in->max_clauses + 31) / 32 * 4 + 16;
  static PerDevice attr;
  attr.get([] {
    return (int)cudaFuncSetAttribute(greedy_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     MAXC * 16 + MAXC / 32 * 4 + 16);
  });
  GR_LAUNCH("greedy_small_kernel", (cudaStream_t)s, greedy_small_kernel<<<in->B, 32, smem, (cudaStream_t)s>>>(*in, *out));
  return GR_OK;
}
