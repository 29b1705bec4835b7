"""Planner parity with the reference (`pkg/src/zeroppsim/planner.py`) on CPU: the
CSV table and summary of every golden search space are identical, byte for byte
(fixtures from tests/golden/make_plan_golden.py), plus the measured-cost search."""

import json
import math
from pathlib import Path

import pytest

from paper_2402_03791_b200 import CommCostModel, ConfigError, ModelSpec, ParallelConfig, RecomputeMode
from paper_2402_03791_b200.planner import SearchSpace, engine_memory_model, report, search, search_measured

GOLDEN = json.loads((Path(__file__).parent / "golden" / "plans.json").read_text())


def _space(case):
    kw = {k: tuple(v) for k, v in case["kw"].items()}
    return SearchSpace(model=ModelSpec(**case["model"]), base=ParallelConfig(**case["parallel"]),
                       costs=CommCostModel(**case["costs"]),
                       memory_cap=math.inf if case["cap"] is None else case["cap"], **kw)


@pytest.mark.parametrize("name", sorted(GOLDEN))
def test_plan_matches_reference(name):
    case = GOLDEN[name]
    csv_text, summary = report(search(_space(case)))
    assert summary == case["summary"]
    assert csv_text == case["csv"]


def test_ac8_cap_sweep_monotone():
    """Acceptance AC8 (test_acceptance.py:247-273): best time never worsens as the cap grows."""
    times = [json.loads(json.dumps(GOLDEN[f"ac8_cap{c}"]["summary"])) for c in (10, 16, 24, 48, 96, 1024, None)]
    vals = [float(s.split("time=")[1].split()[0].rstrip(")")) if s.startswith("best") else math.inf for s in times]
    assert all(b <= a for a, b in zip(vals, vals[1:]))


def test_search_space_validation():
    m = ModelSpec(num_layers=4, hidden_size=8, seq_len=4)
    with pytest.raises(ConfigError):
        SearchSpace(m, ParallelConfig(pp_size=3, dp_size=1, microbatches=3, unit_size=3), CommCostModel(1.0, 1.0))
    with pytest.raises(ConfigError):
        SearchSpace(m, ParallelConfig(pp_size=2, dp_size=1, microbatches=2, unit_size=2), CommCostModel(1.0, 1.0),
                    memory_cap=0)


def test_search_measured_keeps_default_order_and_uses_engine_memory():
    """Measured costs re-time the default-cost order; engine memory fields change peaks."""
    from paper_2402_03791_b200.engine import GPTSpec
    spec = GPTSpec.gpt_6p2b()
    model = ModelSpec(num_layers=32, hidden_size=4096, seq_len=2048)
    fitted, k = engine_memory_model(spec, model)
    fitted = ModelSpec(**{**fitted.__dict__, "t_forward": 2.6, "t_input_grad": 3.1, "t_weight_grad": 2.4,
                          "t_optstep": 1.1})
    base = ParallelConfig(pp_size=2, dp_size=4, microbatches=16, unit_size=8, stages_per_device=2)
    space = SearchSpace(model=model, base=base, costs=CommCostModel(intra_node_bandwidth=4e8,
                                                                     inter_node_bandwidth=5e7),
                        memory_cap=180e9, unit_sizes=(4, 8, 16), stage_counts=(1, 2, 4),
                        recompute_modes=(RecomputeMode.NONE,))
    plan = search_measured(space, fitted, space.costs, optimizer_state_multiplier=k)
    assert len(plan.rows) == 3 * 3 * 2 and plan.best is not None
    assert all(r.time > 0 for r in plan.rows)
    # engine memory: static 16 B/param of optimizer state per (P*D) shard shows up in every peak
    assert min(r.peak_mem for r in plan.rows) > 8.0 * 2 * spec.num_params() / 8 * 0.9
