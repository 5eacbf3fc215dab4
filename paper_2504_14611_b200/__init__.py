"""B200-native (sm_100a) J-DOB hot path (arXiv 2504.14611).

Public API (thin binding over the C ABI in include/jdob.h, kernels in csrc/):
  DeviceBatch, solve_batch, solve_batch_modes, stats, eval_plans, plan_partition, bruteforce, bf_space_size,
  HostBuffers, solve_batch_host, and the multi-GPU helpers in .dist.
"""
from ._binding import (  # noqa: F401
    DeviceBatch, HostBuffers, JdobError, bf_space_size, bruteforce, eval_plans, lib, plan_partition, solve_batch,
    shared_params,
    solve_batch_host, solve_batch_modes, solve_grouped, release_pool, stats, EXPORTED, LIB_PATH,
    MODE_FULL, MODE_LC, MODE_NO_EDGE_DVFS, MODE_BINARY, SPACE_GENERAL, SPACE_IDENTICAL,
    ST_OK, ST_LOCAL_INFEASIBLE, ST_REQUIRE, ST_BADPARAM, ST_BADMODEL, ST_TOOBIG, STATS_FIELDS, MAX_M, MAX_N, MAX_K,
)

__version__ = "0.1.0"
