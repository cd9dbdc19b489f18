"""B200-native batched trace-driven simulator (Maya / dltsim hot path).

Public API (reference-shaped, see api.py):
    simulate, compute_mfu, GpuPipelineEvaluator, evaluate_space,
    evaluate_space_distributed, SimDeadlockError
Lower level: engine.Engine (C ABI in include/maya_b200.h), rawtrace.RawJob,
workload.generate_job (native trace generator).
"""

__version__ = "0.1.0"

from .api import (GpuPipelineEvaluator, SimDeadlockError, compute_mfu,  # noqa: F401
                  evaluate_space, evaluate_space_distributed, simulate)
