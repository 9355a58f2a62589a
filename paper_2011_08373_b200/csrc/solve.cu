// solve.cu -- gr_solve: the Solve step of Alg. 1 with the
// paper's two strategies.
//
//   GR_STRATEGY_MAXSAT: the (weighted) partial-MaxSAT optimum = gr_solve_pms.
//   GR_STRATEGY_MHS:    Johnson's greedy mhs over phi+ (gr_mhs_greedy); every
//                       instance whose greedy set breaks phi- ("results in
//                       unsatisfiability") falls back to the
//                       MaxSAT solver, i.e. gets the gr_solve_pms result.
//   GR_STRATEGY_MHS_FINAL: the mhs strategy's final "single query to a MaxSAT
//                       solver": the greedy answer, then the
//                       MaxSAT optimum; fell_back = the query changed it.
// With weights, the cost of a greedy answer is its weight (the greedy itself
// is unweighted, as in the paper's mhs strategy).
#include "common.cuh"

int gr_exact_solve_selected(const gr_batch *in, gr_result *out, void *ws, size_t ws_bytes,
                            gr_stream_t s, const int32_t *sel, int sel_val);
uint64_t *gr_exact_scratch(const gr_batch *in, void *ws);

namespace {
__global__ void after_greedy_kernel(gr_batch in, gr_result out, int32_t *fell_back) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= in.B) return;
  const int st = out.status[b];
  if (fell_back) fell_back[b] = st == GR_SAT_NEG_VIOLATED;
  if (out.decided) out.decided[b] = 0;
  if (in.w && st == GR_SAT) {  // weight of the greedy set
    u64 c = 0;
    for (int t = 0; t < in.W; t++) {
      u64 a = out.assign[(size_t)b * in.W + t];
      while (a) {
        const int i = __ffsll((long long)a) - 1;
        a &= a - 1;
        c += in.w[(size_t)b * in.wstride + 64 * t + i];
      }
    }
    out.cost[b] = c;
  }
}
// GR_STRATEGY_MHS_FINAL, before the MaxSAT query: the greedy answer's cost
// (its weight with weights; UINT64_MAX when it broke phi- or was not SAT)
__global__ void greedy_cost_kernel(gr_batch in, gr_result out, uint64_t *gcost) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= in.B) return;
  u64 c = ~0ull;
  if (out.status[b] == GR_SAT) {
    c = 0;
    for (int t = 0; t < in.W; t++)
      for (u64 a = out.assign[(size_t)b * in.W + t]; a; a &= a - 1)
        c += in.w ? in.w[(size_t)b * in.wstride + 64 * t + __ffsll((long long)a) - 1] : 1u;
  }
  gcost[b] = c;
}
// after it: fell_back[b] = 1 where the query changed the answer -- the greedy
// set broke phi-, or the optimum is cheaper than the greedy set
__global__ void final_flag_kernel(gr_batch in, gr_result out, const uint64_t *gcost,
                                  int32_t *fell_back) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= in.B) return;
  fell_back[b] = gcost[b] == ~0ull || (out.status[b] == GR_SAT && out.cost[b] < gcost[b]);
}
}  // namespace

extern "C" int gr_solve(const gr_batch *in, int strategy, gr_result *out, int32_t *fell_back,
                        void *ws, size_t ws_bytes, gr_stream_t s) {
  if (!in || !out) { gr_set_error("null argument"); return GR_EINVAL; }
  if (strategy == GR_STRATEGY_MAXSAT) {
    if (fell_back) GR_CUDA(cudaMemsetAsync(fell_back, 0, sizeof(int32_t) * in->B, (cudaStream_t)s));
    return gr_solve_pms(in, out, ws, ws_bytes, s);
  }
  if (strategy == GR_STRATEGY_MHS_FINAL) {
    // the mhs strategy's "single query to a MaxSAT solver ... to ensure that
    // the number of b_i's being set to true is the minimum":
    // the greedy answer, then the (weighted) partial-MaxSAT optimum for every
    // instance; fell_back marks where the query changed the answer
    if (!ws || ws_bytes < gr_workspace_bytes(in, 0)) { gr_set_error("workspace too small"); return GR_EWORKSPACE; }
    int rc = gr_mhs_greedy(in, out, ws, ws_bytes, s);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)s;
    uint64_t *gcost = gr_exact_scratch(in, ws);
    const int g = (in->B + 255) / 256;
    GR_LAUNCH("greedy_cost_kernel", st, greedy_cost_kernel<<<g, 256, 0, st>>>(*in, *out, gcost));
    if ((rc = gr_solve_pms(in, out, ws, ws_bytes, s))) return rc;
    if (fell_back) GR_LAUNCH("final_flag_kernel", st, final_flag_kernel<<<g, 256, 0, st>>>(*in, *out, gcost, fell_back));
    return GR_OK;
  }
  if (strategy != GR_STRATEGY_MHS) { gr_set_error("unknown strategy"); return GR_EINVAL; }
  int rc = gr_mhs_greedy(in, out, ws, ws_bytes, s);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)s;
  GR_LAUNCH("after_greedy_kernel", st,
            after_greedy_kernel<<<(in->B + 255) / 256, 256, 0, st>>>(*in, *out, fell_back));
  // MaxSAT fallback for the instances whose mhs breaks phi- 
  return gr_exact_solve_selected(in, out, ws, ws_bytes, s, out->status, GR_SAT_NEG_VIOLATED);
}
