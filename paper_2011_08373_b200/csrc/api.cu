// api.cu -- error plumbing, version, workspace query of libgrsolve.
#include <string>

#include "common.cuh"

static thread_local std::string g_err;

void gr_set_error(const std::string &msg) { g_err = msg; }

int gr_cuda_fail(cudaError_t e, const char *where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return GR_ECUDA;
}

extern "C" size_t gr_workspace_bytes_exact(const gr_batch *in);

extern "C" const char *gr_last_error(void) { return g_err.c_str(); }

extern "C" const char *gr_version(void) { return "grsolve 0.1 sm_100a"; }

extern "C" size_t gr_workspace_bytes(const gr_batch *in, int which) {
  if (!in || in->B < 1 || (in->W != 1 && in->W != 2)) return 0;
  if (which == 0 || which == 1) return gr_workspace_bytes_exact(in);
  if (which == 2) return 256;  // gr_mhs_greedy needs no scratch
  return 0;
}
