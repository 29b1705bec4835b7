"""simulate() / render_timeline parity with the reference (fixtures from make_sim_golden.py).

Everything is compared bit-for-bit: float fields through repr(), per-task start/end
times and memory traces through sha256, rendered documents as exact strings.
"""

import hashlib
import json
import logging
import warnings
from pathlib import Path

import pytest

import paper_2402_03791_b200 as Z
from paper_2402_03791_b200.render import RenderFormat, chrome_trace, render_timeline
from paper_2402_03791_b200.simulation import SimulationDeadlock, bubble_count, simulate

CASES = json.loads((Path(__file__).parent / "golden" / "simulation.json").read_text())


def _h(s: str) -> str:
    return hashlib.sha256(s.encode()).hexdigest()[:32]


def _build(case):
    m = Z.ModelSpec(**case["model"])
    pk = dict(case["parallel"])
    pk["hybrid_mode"] = Z.HybridMode(pk.get("hybrid_mode", "dp_outer"))
    pk["recompute"] = Z.RecomputeMode(pk.get("recompute", "none"))
    c = Z.ParallelConfig(**pk)
    pl = Z.make_placement(c, m)
    costs = Z.CommCostModel(**case["costs"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        s = Z.generate(m, c, pl, Z.ScheduleVariant(case["variant"]))
    return m, c, pl, costs, s


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_simulate_matches_reference(case):
    m, c, pl, costs, s = _build(case)
    r = simulate(s, m, c, pl, costs)
    assert repr(r.makespan) == case["makespan"]
    assert [repr(x) for x in r.per_device_busy] == case["busy"]
    assert [repr(x) for x in r.per_device_idle] == case["idle"]
    assert [repr(x) for x in r.peak_mem] == case["peak_mem"]
    assert [[repr(b.total), repr(b.weights), repr(b.activations), repr(b.gradients), repr(b.optimizer)]
            for b in r.peak_components] == case["components"]
    assert repr(r.comm_bytes_intra) == case["intra"] and repr(r.comm_bytes_inter) == case["inter"]
    assert [repr(x) for x in r.bubble_ratios] == case["bubble_ratios"]
    times = " ".join(f"{t.task_id}:{r.task_times[t][0]!r}:{r.task_times[t][1]!r}"
                     for lst in s.per_device for t in lst)
    assert _h(times) == case["times_sha"]
    assert _h(repr(r.mem_trace)) == case["mem_sha"]
    if "ascii" in case:
        logging.disable(logging.WARNING)
        try:
            assert render_timeline(r, s, RenderFormat.ASCII) == case["ascii"]
            assert render_timeline(r, s, "svg") == case["svg"]
        finally:
            logging.disable(logging.NOTSET)


def test_bubble_count_and_errors():
    case = next(c for c in CASES if c["name"] == "C1/inf")
    m, c, pl, costs, s = _build(case)
    r = simulate(s, m, c, pl, costs)
    assert bubble_count(r) == max(r.per_device_idle)  # unit-cost tasks: slot = 1
    with pytest.raises(Z.ConfigError):
        render_timeline(r, s, "png")
    trace = json.loads(chrome_trace(r, s, time_unit_us=1.0))
    assert sum(1 for e in trace["traceEvents"] if e["ph"] == "X") == len(list(s.tasks()))


def test_simulate_deadlock_and_missing():
    case = next(c for c in CASES if c["name"] == "C1/inf")
    m, c, pl, costs, s = _build(case)
    lst = s.per_device[0]
    f = [t for t in lst if t.kind is Z.TaskKind.F]
    # swap two dependent forwards on device 0 of stages 0 -> 2: F(s2,m0) before F(s0,m0) is a cycle
    bad = list(lst)
    i, j = bad.index(f[0]), bad.index(next(t for t in f if t.stage == 2 and t.microbatch == 0))
    bad[i], bad[j] = bad[j], bad[i]
    s2 = Z.Schedule(s.variant, [bad] + s.per_device[1:], s.edges)
    with pytest.raises(SimulationDeadlock) as ei:
        simulate(s2, m, c, pl, costs)
    assert ei.value.frontier
    s3 = Z.Schedule(s.variant, [lst[1:]] + s.per_device[1:], s.edges)
    with pytest.raises(ValueError, match="missing from schedule"):
        simulate(s3, m, c, pl, costs)
