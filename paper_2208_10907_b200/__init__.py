"""B200-native dependency-free H2-ULV hot path (arXiv 2208.10907).

Python mirror of the reference's proj/include API for the hot path
(RunConfig / Pipeline, report.hpp:13-99) over the C-ABI in include/h2g.h,
implemented by the in-tree sm_100a library libh2g.so. There is no CPU
fallback: importing works anywhere, but every compute call raises if the
library or a CUDA device is missing.
"""
from ._lib import (Comm, H2GError, Problem, generate_points, gloo_allgather, lib,  # noqa: F401
                   lib_path, nccl_unique_id, partition_range)
from .pipeline import RunConfig, Pipeline, make_cloud, run_pipeline  # noqa: F401

__all__ = ["H2GError", "Problem", "RunConfig", "Pipeline", "make_cloud", "run_pipeline", "lib",
           "lib_path", "Comm", "nccl_unique_id", "partition_range", "gloo_allgather", "generate_points"]
