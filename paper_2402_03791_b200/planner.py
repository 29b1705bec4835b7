"""Configuration search under a per-device memory cap.

Restates the reference planner (`pkg/src/zeroppsim/planner.py:38-189`): fix the
cluster shape (P, D, n) and the batch split (B micro-batches), sweep unit size U,
stages per device V, recompute and the outer hybrid mode; generate + validate +
simulate every candidate and rank feasible ones by (time, peak memory, U, V,
recompute, mode) and infeasible ones by (peak memory, time, ...).  ``search`` /
``report`` reproduce the reference bit-for-bit (tests/golden/plans.json).

The engine extension is :func:`search_measured`: the B200 costs come from a
measured step (:func:`engine.timeline.calibrate`) and the memory model from the
engine's real buffers (:func:`engine_memory_model`).  Because the generated order
depends on the cost ratios, each candidate is generated
with the DEFAULT abstract costs -- the order the engine executes and the
reference pins -- and only its timing is re-simulated with the measured costs
(``engine.timeline.predict`` semantics).
"""

from __future__ import annotations

import csv
import dataclasses
import functools
import io
import math
import warnings
from dataclasses import dataclass

from .config import CommCostModel, ConfigError, HybridMode, ModelSpec, ParallelConfig, RecomputeMode, make_placement
from .schedules import generate
from .simulation import simulate
from .tasks import Schedule, ScheduleVariant, TaskKind
from .validation import validate

__all__ = ["SearchSpace", "PlanRow", "PlanResult", "search", "report", "search_measured",
           "engine_memory_model"]


def _divisors(n: int) -> tuple[int, ...]:
    return tuple(d for d in range(1, n + 1) if n % d == 0)


@dataclass(frozen=True)
class SearchSpace:
    """Candidate grid around ``base`` (planner.py:38-79): U defaults to every
    divisor of B, V to every divisor of L/P; ``memory_cap`` in the model's memory unit."""

    model: ModelSpec
    base: ParallelConfig
    costs: CommCostModel
    memory_cap: float = math.inf
    unit_sizes: tuple[int, ...] | None = None
    stage_counts: tuple[int, ...] | None = None
    recompute_modes: tuple[RecomputeMode, ...] = (RecomputeMode.NONE, RecomputeMode.FULL)
    hybrid_modes: tuple[HybridMode, ...] = (HybridMode.DP_OUTER, HybridMode.ZERO1_OUTER)

    def __post_init__(self):
        if self.memory_cap <= 0:
            raise ConfigError("memory_cap must be > 0")
        if self.model.num_layers % self.base.pp_size != 0:
            raise ConfigError("num_layers must be divisible by pp_size")

    def resolved_unit_sizes(self) -> tuple[int, ...]:
        return self.unit_sizes if self.unit_sizes is not None else _divisors(self.base.microbatches)

    def resolved_stage_counts(self) -> tuple[int, ...]:
        if self.stage_counts is not None:
            return self.stage_counts
        return _divisors(self.model.num_layers // self.base.pp_size)

    def grid_size(self) -> int:
        return (len(self.resolved_unit_sizes()) * len(self.resolved_stage_counts())
                * len(self.recompute_modes) * len(self.hybrid_modes))

    def candidates(self):
        for u in self.resolved_unit_sizes():
            for v in self.resolved_stage_counts():
                for rec in self.recompute_modes:
                    for mode in self.hybrid_modes:
                        yield dataclasses.replace(self.base, unit_size=u, stages_per_device=v,
                                                  recompute=rec, hybrid_mode=mode)


@dataclass(frozen=True)
class PlanRow:
    unit_size: int
    stages_per_device: int
    recompute: RecomputeMode
    hybrid_mode: HybridMode
    time: float
    peak_mem: float
    feasible: bool

    def _knobs(self):
        return (self.unit_size, self.stages_per_device, self.recompute.value, self.hybrid_mode.value)


@dataclass(frozen=True)
class PlanResult:
    """Feasible rows first by (time, peak, knobs), then infeasible by (peak, time, knobs)."""

    rows: tuple[PlanRow, ...]
    best: PlanRow | None
    memory_cap: float

    @property
    def feasible_rows(self) -> tuple[PlanRow, ...]:
        return tuple(r for r in self.rows if r.feasible)

    @property
    def min_memory_row(self) -> PlanRow:
        return min(self.rows, key=lambda r: (r.peak_mem, r.time, r.unit_size))


def _generate_checked(model: ModelSpec, cfg: ParallelConfig):
    placement = make_placement(cfg, model)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")  # recompute=full with V=1 is a legal grid point (it warns)
        sched = generate(model, cfg, placement, ScheduleVariant.ZEROPP)
    bad = validate(sched, placement, cfg)
    if bad:  # a generator bug, never a user error
        raise RuntimeError(f"generated candidate failed validation: {bad[0]}")
    return placement, sched


@functools.lru_cache(maxsize=4096)
def _evaluate(model: ModelSpec, cfg: ParallelConfig, costs: CommCostModel) -> tuple[float, float]:
    placement, sched = _generate_checked(model, cfg)
    res = simulate(sched, model, cfg, placement, costs)
    return res.makespan, max(res.peak_mem)


def _rank(rows: list[PlanRow], cap: float) -> PlanResult:
    ok = sorted((r for r in rows if r.feasible), key=lambda r: (r.time, r.peak_mem) + r._knobs())
    bad = sorted((r for r in rows if not r.feasible), key=lambda r: (r.peak_mem, r.time) + r._knobs())
    return PlanResult(tuple(ok + bad), ok[0] if ok else None, cap)


def search(space: SearchSpace) -> PlanResult:
    """Evaluate the whole grid with the reference cost / memory model (planner.py:130-157)."""
    rows = []
    for cfg in space.candidates():
        t, peak = _evaluate(space.model, cfg, space.costs)
        rows.append(PlanRow(cfg.unit_size, cfg.stages_per_device, cfg.recompute, cfg.hybrid_mode, t, peak,
                            peak <= space.memory_cap))
    return _rank(rows, space.memory_cap)


def _fmt(x: float) -> str:
    return f"{x:.10g}"


def report(plan: PlanResult) -> tuple[str, str]:
    """(CSV table, one-line summary), as planner.py:163-189 renders them."""
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(["U", "V", "recompute", "mode", "time", "peak_mem", "feasible"])
    for r in plan.rows:
        w.writerow([r.unit_size, r.stages_per_device, r.recompute.value, r.hybrid_mode.value, _fmt(r.time),
                    _fmt(r.peak_mem), int(r.feasible)])
    cap = "unbounded" if math.isinf(plan.memory_cap) else _fmt(plan.memory_cap)
    if plan.best is not None:
        b = plan.best
        summary = (f"best candidate: U={b.unit_size} V={b.stages_per_device} recompute={b.recompute.value} "
                   f"mode={b.hybrid_mode.value} time={_fmt(b.time)} peak_mem={_fmt(b.peak_mem)} "
                   f"(cap={cap}; {len(plan.feasible_rows)}/{len(plan.rows)} candidates feasible)")
    else:
        m = plan.min_memory_row
        summary = (f"no feasible candidate under cap={cap}; closest is U={m.unit_size} V={m.stages_per_device} "
                   f"recompute={m.recompute.value} mode={m.hybrid_mode.value} with peak_mem={_fmt(m.peak_mem)} "
                   f"(time={_fmt(m.time)})")
    return buf.getvalue(), summary


# --------------------------------------------------------------------------- engine extension
def engine_memory_model(spec, model: ModelSpec) -> tuple[ModelSpec, float]:
    """ModelSpec whose memory fields are the engine's real bytes, and the matching
    optimizer-state multiplier k (``ParallelConfig.optimizer_state_multiplier``).

    * weights: bf16 stage parameters, ``weight_mem_per_layer`` = per-layer parameter
      count x 2 B (GPT 12h^2 + 13h; LLaMA 4h^2 + 3h*ffn + 2h);
    * activations: the F->B stash per layer per micro-batch --
      GPT: x, xn1, qkv(3h), o, x1, xn2, u(4h), g(4h) bf16 + 4 fp32 row stats + lse;
      LLaMA: x, xn1, qkv, o, x1, xn2, gu(2f), a(f) bf16 + 2 fp32 row stats + lse;
    * optimizer: fp32 master + exp_avg + exp_avg_sq + grad shard = 16 B per parameter
      = 8x the bf16 shard the reference charges k times (`simulation.py:171-172`).
    """
    h, T, H = spec.hidden, spec.tokens_per_microbatch, spec.heads
    if spec.llama:
        params = 4 * h * h + 3 * h * spec.ffn + 2 * h
        act = T * 2 * (7 * h + 3 * spec.ffn) + T * 4 * 2 + H * T * 4
    else:
        params = 12 * h * h + 13 * h
        act = T * 2 * (16 * h) + T * 4 * 4 + H * T * 4
    fitted = dataclasses.replace(model, weight_mem_per_layer=float(2 * params),
                                 act_mem_per_layer_per_microbatch=float(act))
    return fitted, 8.0


def _order_with_default_costs(model: ModelSpec) -> ModelSpec:
    return dataclasses.replace(model, t_forward=1.0, t_input_grad=1.0, t_weight_grad=1.0, t_optstep=0.0)


def search_measured(space: SearchSpace, fitted: ModelSpec, costs: CommCostModel,
                    optimizer_state_multiplier: float | None = None) -> PlanResult:
    """Rank the grid by predicted B200 step time.

    ``fitted`` carries measured per-layer costs (ms) and, typically, the engine's
    memory fields (:func:`engine_memory_model`); ``costs`` the fitted bandwidths.
    Each candidate's task ORDER is generated with the default abstract costs (what
    the engine runs); its times are then simulated with ``fitted`` costs."""
    order_model = _order_with_default_costs(fitted)
    rows = []
    for cfg in space.candidates():
        if optimizer_state_multiplier is not None:
            cfg = dataclasses.replace(cfg, optimizer_state_multiplier=optimizer_state_multiplier)
        placement, sched = _generate_checked(order_model, cfg)
        res = simulate(_recost(sched, fitted, placement), fitted, cfg, placement, costs)
        peak = max(res.peak_mem)
        rows.append(PlanRow(cfg.unit_size, cfg.stages_per_device, cfg.recompute, cfg.hybrid_mode,
                            res.makespan, peak, peak <= space.memory_cap))
    return _rank(rows, space.memory_cap)


def _recost(sched: Schedule, fitted: ModelSpec, placement) -> Schedule:
    """The same tasks in the same order with ``fitted`` compute costs (bytes unchanged)."""
    per_layer = {TaskKind.F: fitted.t_forward, TaskKind.R: fitted.t_forward,
                 TaskKind.B: fitted.t_input_grad, TaskKind.W: fitted.t_weight_grad}

    def cost(t):
        if t.kind in per_layer:
            return per_layer[t.kind] * placement.layers_in_stage(t.stage)
        if t.kind is TaskKind.OPT:
            return fitted.t_optstep * sum(placement.layers_in_stage(s) for s in placement.device_stages(t.device))
        return t.cost

    remap = {t: dataclasses.replace(t, cost=cost(t)) for t in sched.tasks()}
    return Schedule(sched.variant, [[remap[t] for t in lst] for lst in sched.per_device],
                    {(remap[a], remap[b]) for a, b in sched.edges})
