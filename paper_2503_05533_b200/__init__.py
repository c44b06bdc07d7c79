"""B200-native (sm_100a) hot path of the MPML method of arXiv 2503.05533.

The product is the C-ABI library ``libmlmc.so`` (include/mlmc.h) built from
``csrc/`` by :mod:`paper_2503_05533_b200.build`; :mod:`.api` is its thin
Python binding.  There is no CPU fallback.
"""
from .api import (Context, precision, mlmc_plan_levels, mlmc_sample_level, mlmc_sample_level_async,  # noqa: F401
                  mlmc_adaptive_run, mlmc_eps_schedule, mlmc_optimal_samples, mlmc_kl_modes, mlmc_debug_field,
                  mlmc_workspace_bytes)
