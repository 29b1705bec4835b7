"""B200-native ZeroPP training engine.

The host API mirrors the reference package ``zeroppsim``
(`pkg/src/zeroppsim/__init__.py:10-54`) for the hot-path subset - configure,
generate, validate, export - and adds :func:`execute`, the real-hardware
replacement for the reference's ``simulate`` (`simulation.py:90-158`).  The
GPU work runs in ``libzpp.so`` (hand-written sm_100a kernels + NCCL) through a
plain C ABI (`include/zpp.h`); there is no CPU fallback.
"""

from .config import (
    CommCostModel,
    ConfigError,
    HybridMode,
    ModelSpec,
    ParallelConfig,
    Placement,
    RecomputeMode,
    load_config,
    make_placement,
)
from .costmodel import (
    TABLE_METHODS,
    CostReport,
    Method,
    bubble_formula,
    crossover,
    figure1_curve,
    memory_formula,
    table2_row,
    tp_comm_volume,
    zeropp_comm_volume,
)
from .schedules import apply_recompute, build_dependency_edges, expected_edges, generate
from .tasks import (
    Schedule,
    ScheduleVariant,
    Task,
    TaskKind,
    export_text,
    schedule_from_json,
    schedule_to_json,
)
from .validation import FuzzSummary, Violation, ViolationKind, fuzz_check, validate
from .simulation import (
    MemoryBreakdown,
    SimResult,
    SimulationDeadlock,
    bubble_count,
    comm_volume,
    peak_memory,
    simulate,
)
from .render import RenderFormat, chrome_trace, render_timeline
from .planner import PlanResult, PlanRow, SearchSpace, report, search, search_measured

__version__ = "0.1.0"

__all__ = [
    "CommCostModel", "ConfigError", "FuzzSummary", "HybridMode", "ModelSpec",
    "ParallelConfig", "Placement", "RecomputeMode", "Schedule", "ScheduleVariant",
    "Task", "TaskKind", "Violation", "ViolationKind", "apply_recompute",
    "build_dependency_edges", "execute", "expected_edges", "export_text", "fuzz_check",
    "generate", "load_config", "make_placement", "schedule_from_json",
    "schedule_to_json", "validate", "__version__",
    "MemoryBreakdown", "SimResult", "SimulationDeadlock", "bubble_count", "comm_volume",
    "peak_memory", "simulate", "RenderFormat", "chrome_trace", "render_timeline",
    "PlanResult", "PlanRow", "SearchSpace", "report", "search", "search_measured",
    "TABLE_METHODS", "CostReport", "Method", "bubble_formula", "crossover", "figure1_curve",
    "memory_formula", "table2_row", "tp_comm_volume", "zeropp_comm_volume",
]


def execute(*args, **kwargs):
    """Run one ZeroPP training step on this rank's GPU (see :mod:`.engine`)."""
    from .engine import execute as _execute
    return _execute(*args, **kwargs)
