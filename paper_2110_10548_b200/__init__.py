"""redsynth-b200: B200-native executor for the reduction programs of P²
(arXiv 2110.10548). Host planner (C++, reference API) + sm_100a P2P kernels
behind a C-ABI; see DESIGN.md."""
from . import planner  # noqa: F401

__all__ = ["planner", "executor"]
