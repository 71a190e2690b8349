"""B200-native HHL state-vector hot path (arXiv 2402.08136).

The product is the C-ABI library libhhlsv.so (include/sv.h) built from csrc/ for
sm_100a; `sv` is its thin ctypes binding with the same names. Nothing here imports
the test oracle (oracle/), and there is no CPU fallback.
"""
from .sv import (EXPORTS, HHLProgram, Program, State, SVError, comm_bench, hhl_plan_size,  # noqa: F401
                 hhl_schedule_dump, hhl_solve, load, nccl_unique_id, schedule_dump, trim_memory)

__all__ = ["State", "Program", "HHLProgram", "SVError", "hhl_solve", "hhl_plan_size", "hhl_schedule_dump", "load", "nccl_unique_id",
           "comm_bench", "trim_memory", "EXPORTS"]
