"""Measured-timeline adapter: executed steps as reference-shaped ``SimResult``s.

SURVEY.md section 8(f) row 2.  ``measured_result`` turns the CUDA-event task times
of :func:`execute` (per rank, ms from the step's first event, each task's start
taken AFTER its stream waits so P2P / AG waits count as idle, not busy) into the
reference's result type (`pkg/src/zeroppsim/simulation.py:53-77`): one lane per
pipeline device, gathered from the z = 0 rank of every pipeline rank.  Busy / idle /
bubble ratios therefore mean what they mean for ``simulate``; ``peak_mem`` is the
reference memory model evaluated on the measured times (its component breakdown
and trace stay consistent), while the allocator's real peak per device is in
``extras["peak_mem_measured"]``.  Extras also carry loss, tokens/s, MFU and
exposed comm, the superset SURVEY.md section 8(b) asks of ``execute``.

``calibrate`` fits the abstract per-layer costs (ms) and an effective ZeRO
bandwidth from a measured step; ``predict`` re-simulates the EXECUTED schedule
with those costs (task order kept: regenerating with non-default costs changes
the order), so measured and predicted makespan / bubble can
be compared and both rendered with :func:`paper_2402_03791_b200.render_timeline`.
"""

from __future__ import annotations

import dataclasses
import statistics

import torch

from ..config import CommCostModel, ModelSpec
from ..simulation import SimResult, simulate, summarize
from ..tasks import Schedule, TaskKind

__all__ = ["measured_result", "calibrate", "predict", "model_flops_per_token"]


def model_flops_per_token(spec) -> float:
    """Model FLOPs per token (GPT or LLaMA), attention at full s^2."""
    return spec.flops_per_token()


def measured_result(runtime, res, gather: bool = True, peak_flops: float = 2.25e15) -> SimResult:
    """Reference-shaped result of the step ``res`` (from ``execute`` with a
    ``timeline=True`` runtime).  With ``gather`` and a multi-rank job every rank
    must call it (collective); all ranks get the whole-job result."""
    if not res.task_times:
        raise ValueError("no task times: build the Runtime with timeline=True")
    rt = runtime
    mine = [(t.task_id, s, e) for t, (s, e) in res.task_times.items()]
    peak_alloc = float(torch.cuda.max_memory_allocated(rt.dev))
    local = {"p": rt.p, "z": rt.z, "node": rt.node, "times": mine, "peak": peak_alloc, "step_ms": res.step_ms,
             "loss_sum": float(res.loss_sum.item()), "tokens": res.tokens,
             "exposed": res.exposed_comm_ms or 0.0, "p2p": res.p2p_wait_ms or 0.0}
    if gather and rt.world > 1:
        import torch.distributed as dist
        parts = [None] * rt.world
        dist.all_gather_object(parts, local)
    else:
        parts = [local]
    sched: Schedule = rt.sched
    by_id = {t.task_id: t for t in sched.tasks()}
    times = {}
    peaks = [0.0] * sched.num_devices
    for part in parts:
        peaks[part["p"]] = max(peaks[part["p"]], part["peak"])
        if part["z"] != 0 or part["node"] != 0:
            continue
        for tid, s, e in part["times"]:
            times[by_id[tid]] = (s, e)
    cfg, spec = rt.cfg, rt.spec
    tokens_job = cfg.inter_node_dp * cfg.dp_size * cfg.microbatches * spec.tokens_per_microbatch
    step_ms = max(p["step_ms"] for p in parts)
    loss_sum = sum(p["loss_sum"] for p in parts)
    tok_s = tokens_job / (step_ms / 1e3)
    extras = {
        "loss": loss_sum / tokens_job,
        "step_ms": step_ms,
        "tokens_per_s": tok_s,
        "mfu": tok_s * model_flops_per_token(spec) / (peak_flops * rt.world),
        "exposed_comm_ms": max(p["exposed"] for p in parts),
        "p2p_wait_ms": max(p["p2p"] for p in parts),
        "peak_mem_measured": peaks,
        "time_unit": "ms",
    }
    if len(times) != len(by_id):
        extras["partial"] = True  # gather=False on a multi-device job: only this lane
        sub = Schedule(sched.variant, [lst if any(t in times for t in lst) else [] for lst in sched.per_device],
                       {(a, b) for a, b in sched.edges if a in times and b in times})
        return summarize(sub, rt.model, cfg, rt.pl, times, extras)
    return summarize(sched, rt.model, cfg, rt.pl, times, extras)


def calibrate(measured: SimResult, sched: Schedule, model: ModelSpec, placement) -> tuple[ModelSpec, CommCostModel]:
    """Per-layer F/B/W/OPT costs (median ms per layer) and an effective intra-node
    bandwidth (bytes/ms) fitted to a measured step; the inter-node bandwidth is fitted
    to the outer tasks (AR_GRAD / RS_GRAD_INTER / AG_PARAM_INTER) when they moved bytes."""
    per_layer = {k: [] for k in (TaskKind.F, TaskKind.B, TaskKind.W, TaskKind.R)}
    opt, comm_bw, inter_bw = [], [], []
    for t, (s, e) in measured.task_times.items():
        if t.kind in per_layer and t.stage is not None:
            per_layer[t.kind].append((e - s) / placement.layers_in_stage(t.stage))
        elif t.kind is TaskKind.OPT:
            opt.append((e - s) / max(1, sum(placement.layers_in_stage(st)
                                          for st in placement.device_stages(t.device))))
        elif t.is_comm and t.bytes > 0 and e > s:
            inter = t.kind in (TaskKind.AR_GRAD, TaskKind.RS_GRAD_INTER, TaskKind.AG_PARAM_INTER)
            (inter_bw if inter else comm_bw).append(t.bytes / (e - s))
    med = lambda xs, d: statistics.median(xs) if xs else d  # noqa: E731
    fitted = dataclasses.replace(model, t_forward=med(per_layer[TaskKind.F], model.t_forward),
                                 t_input_grad=med(per_layer[TaskKind.B], model.t_input_grad),
                                 t_weight_grad=med(per_layer[TaskKind.W], model.t_weight_grad),
                                 t_optstep=med(opt, model.t_optstep))
    bw = med(comm_bw, 1e30)
    return fitted, CommCostModel(intra_node_bandwidth=bw, inter_node_bandwidth=med(inter_bw, bw))


def predict(sched: Schedule, fitted: ModelSpec, costs: CommCostModel, cfg, placement) -> SimResult:
    """``simulate`` of the executed order with calibrated costs."""
    def cost(t):
        if t.kind in (TaskKind.F, TaskKind.R):
            return fitted.t_forward * placement.layers_in_stage(t.stage)
        if t.kind is TaskKind.B:
            return fitted.t_input_grad * placement.layers_in_stage(t.stage)
        if t.kind is TaskKind.W:
            return fitted.t_weight_grad * placement.layers_in_stage(t.stage)
        if t.kind is TaskKind.OPT:
            return fitted.t_optstep * sum(placement.layers_in_stage(s) for s in placement.device_stages(t.device))
        return t.cost
    remap = {t: dataclasses.replace(t, cost=cost(t)) for t in sched.tasks()}
    resched = Schedule(sched.variant, [[remap[t] for t in lst] for lst in sched.per_device],
                       {(remap[a], remap[b]) for a, b in sched.edges})
    return simulate(resched, fitted, cfg, placement, costs)
