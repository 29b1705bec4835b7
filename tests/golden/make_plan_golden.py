"""Planner golden fixtures from the REAL reference (`pkg/src/zeroppsim/planner.py`).

Run in the build container only:  python tests/golden/make_plan_golden.py
Writes tests/golden/plans.json: for each search space (the AC8 acceptance space at
its seven memory caps, the reference test_planner small space at three caps, and
the BASELINE C2/C3 shapes) the reference ``report`` CSV text and summary line.
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import zeroppsim as R  # noqa: E402

OUT = Path(__file__).with_name("plans.json")


def spaces():
    ac8_m = dict(num_layers=48, hidden_size=5120, seq_len=1024, bytes_per_element=2)
    ac8_p = dict(pp_size=4, dp_size=8, microbatches=48, unit_size=12, stages_per_device=2, microbatch_samples=4,
                 inter_node_dp=2)
    ac8_c = dict(intra_node_bandwidth=300e9, inter_node_bandwidth=25e9)
    for cap in (10, 16, 24, 48, 96, 1024, None):
        yield f"ac8_cap{cap}", ac8_m, ac8_p, ac8_c, (cap * 2 ** 30 if cap else None), {}
    small_m = dict(num_layers=4, hidden_size=8, seq_len=4, weight_mem_per_layer=64.0)
    small_p = dict(pp_size=2, dp_size=4, microbatches=4, unit_size=2, inter_node_dp=2)
    small_c = dict(intra_node_bandwidth=256.0, inter_node_bandwidth=64.0)
    for cap in (None, 1500.0, 1.0):
        yield f"small_cap{cap}", small_m, small_p, small_c, cap, {}
    c3_m = dict(num_layers=32, hidden_size=4096, seq_len=2048)
    c3_p = dict(pp_size=2, dp_size=4, microbatches=16, unit_size=8, stages_per_device=2)
    yield "c3_b16", c3_m, c3_p, dict(intra_node_bandwidth=400e9, inter_node_bandwidth=50e9), 80 * 2 ** 30, \
        {"stage_counts": (1, 2, 4)}
    c2_m = dict(num_layers=24, hidden_size=2048, seq_len=2048, t_input_grad=1.3, t_weight_grad=0.7)
    yield "c2_costs", c2_m, dict(pp_size=2, dp_size=4, microbatches=16, unit_size=8), \
        dict(intra_node_bandwidth=400e9, inter_node_bandwidth=50e9), None, {"unit_sizes": (2, 4, 8, 16)}


def main():
    out = {}
    for name, m, p, c, cap, kw in spaces():
        space = R.SearchSpace(model=R.ModelSpec(**m), base=R.ParallelConfig(**p), costs=R.CommCostModel(**c),
                              memory_cap=math.inf if cap is None else cap, **kw)
        csv_text, summary = R.report(R.search(space))
        out[name] = {"model": m, "parallel": p, "costs": c, "cap": cap, "kw": {k: list(v) for k, v in kw.items()},
                     "csv": csv_text, "summary": summary}
        print(name, summary)
    OUT.write_text(json.dumps(out, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
