"""grsolve: the Solve step of GPURepair (arXiv 2011.08373) on B200 (sm_100a).

Public API (thin marshalling over libgrsolve.so, include/gr.h):
    DeviceBatch, DeviceResult           device-resident clause batches / results
    solve_pms, mhs_exact, mhs_greedy    the three solvers
    solve                               the composite Solve with the MaxSAT fallback
    solve_pms_mhs, solve_step           PMS + MHS in one launch; + the greedy on a side stream
    StepGraph                           solve_step captured as a CUDA graph (replay per step)
    ExactSession, PairSession           prepare / level / finish for sharded runs (PairSession:
                                        the fused PMS + MHS walk)
    pack_bitmatrix, mhs_greedy_matrix   greedy at scale over a bit matrix
    mhs_greedy_lists                    the same greedy from clause lists alone (no bit matrix)
    greedy_count_shard                  shard hook for the multi-GPU greedy
Seeded synthetic workloads: paper_2011_08373_b200.synth.
"""
from ._native import (  # noqa: F401
    GR_BADINPUT, GR_FLAG_EXHAUSTIVE, GR_FLAG_WEIGHTED_GREEDY, GR_FLAG_NO_PRUNE, GR_SAT, GR_SAT_NEG_VIOLATED, GR_UNSAT, GR_UNSUPPORTED, MHS,
    PMS, GREEDY, DeviceBatch, DeviceBitMatrix, DeviceResult, ExactSession, GrError,
    bitmatrix_ld, greedy_count_shard, lib, mhs_exact, mhs_greedy, mhs_greedy_matrix,
    pack_bitmatrix, solve_pms, version, launch_count, profiler, Profiler, solve,
    GR_STRATEGY_MHS, GR_STRATEGY_MAXSAT, GR_STRATEGY_MHS_FINAL, solve_pms_mhs, GreedyShard, to_host_many, GreedyMatrixResult,
    PairSession, mhs_greedy_lists, solve_step, StepGraph,
)
