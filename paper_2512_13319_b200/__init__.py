"""paper_2512_13319_b200 -- B200-native parallel continuous-time MAP trajectory estimation.

Implements the data-parallel hot path of arXiv 2512.13319 (Razavi,
Garcia-Fernandez, Saerkkae): the parallel associative-scan solution of the
time-discretised Onsager--Machlup / LQT form of continuous-time MAP estimation
(parallel Kalman--Bucy filter + continuous-time RTS smoother, parallel two-filter
smoother, iterated Taylor linearisation), as hand-written sm_100a CUDA kernels
behind the C ABI in ``include/pmap.h``.  This package is the thin Python binding
(argument marshalling only); it fails loudly when ``libpmap.so`` is missing.
"""
from .binding import (MapError, Plan, load_library, map_last_error, map_plan, map_plan_destroy,
                      map_solve_linear, map_solve_linear_cov, map_solve_linear_fine, map_solve_nonlinear, map_sync, map_two_filter,
                      map_version, map_solve_sequential,
                      map_shard_phase, map_shard_payload_bytes, shard_range, batch_range,
                      LIB_PATH)

__all__ = ["MapError", "Plan", "load_library", "map_plan", "map_plan_destroy", "map_solve_linear",
           "map_solve_linear_cov", "map_solve_linear_fine", "map_solve_sequential",
           "map_two_filter", "map_solve_nonlinear", "map_sync", "map_last_error", "map_version", "LIB_PATH",
           "map_shard_phase", "map_shard_payload_bytes", "shard_range", "batch_range"]
