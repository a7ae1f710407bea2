"""B200-native DDM-ELM hot path (arxiv 2406.15959): hand-written sm_100a CUDA kernels behind the
C ABI of include/elmddm.h, with a thin Python layer (argument marshalling + torch.distributed).
"""
from ._lib import ElmddmError, RankWarning, load  # noqa: F401
from .solver import Context, Problem, partition, plan_query, solve  # noqa: F401

__all__ = ["Context", "Problem", "solve", "partition", "plan_query", "load", "ElmddmError", "RankWarning"]
