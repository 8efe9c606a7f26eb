"""B200-native discord search (the prepare + PhiDD/HOTSAX search path of arXiv 1901.00155).

``engine``     ctypes mirror of the reference's run_discovery interface over libtsdd_cuda.so
``parallel``   candidate sharding across ranks and the best-so-far exchange
``workloads``  the five seeded BASELINE.json series
``build``      in-tree build of the native libraries
"""
from .engine import (Context, CudaRuntimeError, DiscordResult, DiscoveryConfig, InfeasibleInputError,  # noqa: F401
                     ParameterError, RunOutcome, ValidationError, check_config, load_library,
                     run_discovery)

__all__ = ["Context", "CudaRuntimeError", "DiscordResult", "DiscoveryConfig", "InfeasibleInputError",
           "ParameterError", "RunOutcome", "ValidationError", "check_config", "load_library",
           "run_discovery"]
