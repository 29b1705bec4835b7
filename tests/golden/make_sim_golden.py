"""Generate simulate()/render fixtures from the REAL reference package.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_sim_golden.py

Writes ``tests/golden/simulation.json``: for each case the model / parallel /
cost configs and the reference ``simulate`` result -- makespan, per-device
busy / idle / peak memory (``repr`` strings, so floats are pinned bit-for-bit),
component peaks, comm bytes, sha256 of every task's ``task_id:start!r:end!r``
and of the memory traces -- plus ``render_timeline`` ASCII and SVG documents for
the small cases.  Cases: the five BASELINE configs,
recompute, ZeRO-1 outer mode, no-overlap, non-uniform task costs, BFPP, and 40
seeded random configs.
"""

from __future__ import annotations

import hashlib
import json
import logging
import random
import sys
import warnings
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import zeroppsim as R  # noqa: E402
from zeroppsim.render import RenderFormat, render_timeline  # noqa: E402

logging.disable(logging.WARNING)
OUT = Path(__file__).with_name("simulation.json")


def _h(s: str) -> str:
    return hashlib.sha256(s.encode()).hexdigest()[:32]


def record(name, model_kw, par_kw, cost_kw, variant="zeropp", render=False):
    m = R.ModelSpec(**model_kw)
    pk = dict(par_kw)
    pk["hybrid_mode"] = R.HybridMode(pk.get("hybrid_mode", "dp_outer"))
    pk["recompute"] = R.RecomputeMode(pk.get("recompute", "none"))
    c = R.ParallelConfig(**pk)
    pl = R.make_placement(c, m)
    costs = R.CommCostModel(**cost_kw)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        s = R.generate(m, c, pl, R.ScheduleVariant(variant))
    r = R.simulate(s, m, c, pl, costs)
    times = " ".join(f"{t.task_id}:{r.task_times[t][0]!r}:{r.task_times[t][1]!r}"
                     for lst in s.per_device for t in lst)
    rec = {
        "name": name, "model": model_kw, "parallel": par_kw, "costs": cost_kw, "variant": variant,
        "makespan": repr(r.makespan),
        "busy": [repr(x) for x in r.per_device_busy],
        "idle": [repr(x) for x in r.per_device_idle],
        "peak_mem": [repr(x) for x in r.peak_mem],
        "components": [[repr(b.total), repr(b.weights), repr(b.activations), repr(b.gradients),
                        repr(b.optimizer)] for b in r.peak_components],
        "intra": repr(r.comm_bytes_intra), "inter": repr(r.comm_bytes_inter),
        "bubble_ratios": [repr(x) for x in r.bubble_ratios],
        "times_sha": _h(times),
        "mem_sha": _h(repr(r.mem_trace)),
    }
    if render:
        rec["ascii"] = render_timeline(r, s, RenderFormat.ASCII)
        rec["svg"] = render_timeline(r, s, RenderFormat.SVG)
    return rec


def main():
    cases = []
    C_FAST = {"intra_node_bandwidth": 1e6, "inter_node_bandwidth": 2.5e5, "per_collective_latency": 0.25}
    C_NOOV = dict(C_FAST, overlap_with_compute=False)
    C_INF = {"intra_node_bandwidth": 1e30, "inter_node_bandwidth": 1e30}
    base = [
        ("C1", dict(num_layers=4, hidden_size=256, seq_len=128),
         dict(pp_size=2, dp_size=2, microbatches=8, unit_size=4, stages_per_device=2), True),
        ("C2", dict(num_layers=24, hidden_size=2048, seq_len=2048),
         dict(pp_size=2, dp_size=4, microbatches=16, unit_size=8, stages_per_device=2), False),
        ("C3", dict(num_layers=32, hidden_size=4096, seq_len=2048),
         dict(pp_size=2, dp_size=4, microbatches=16, unit_size=8, stages_per_device=2), False),
        ("C4", dict(num_layers=32, hidden_size=4096, seq_len=4096),
         dict(pp_size=4, dp_size=2, microbatches=32, unit_size=8, stages_per_device=2), False),
        ("C5", dict(num_layers=40, hidden_size=5120, seq_len=2048),
         dict(pp_size=8, dp_size=1, microbatches=128, unit_size=16, stages_per_device=1), False),
    ]
    for name, mk, pk, small in base:
        for cname, ck in (("inf", C_INF), ("fast", C_FAST), ("nooverlap", C_NOOV)):
            if name == "C3":
                ck = {"intra_node_bandwidth": 4.0e8, "inter_node_bandwidth": 5e7, "per_collective_latency": 0.01,
                      "overlap_with_compute": ck.get("overlap_with_compute", True)} if cname != "inf" else ck
            cases.append(record(f"{name}/{cname}", mk, pk, ck, render=small))
    c1m, c1p = base[0][1], base[0][2]
    cases.append(record("C1/recompute", c1m, dict(c1p, recompute="full"), C_FAST, render=True))
    cases.append(record("C1/zero1", c1m, dict(c1p, inter_node_dp=2, hybrid_mode="zero1_outer"), C_FAST, render=True))
    cases.append(record("C1/dpouter", c1m, dict(c1p, inter_node_dp=2), C_FAST, render=True))
    cases.append(record("C1/costs", dict(c1m, t_forward=1.0, t_input_grad=2.0, t_weight_grad=1.5, t_optstep=0.5),
                        c1p, C_FAST, render=True))
    cases.append(record("C1/bfpp", c1m, c1p, C_FAST, variant="bfpp", render=True))
    cases.append(record("C1/bfpp-inf", c1m, c1p, C_INF, variant="bfpp", render=True))
    rng = random.Random(20240817)
    for i in range(40):
        P = rng.choice((1, 2, 3, 4, 8))
        V = rng.choice((1, 2, 3))
        U = rng.choice((1, 2, 3, 4, 6, 8))
        B = U * rng.choice((1, 2, 3))
        L = P * V * rng.choice((1, 2))
        n = rng.choice((1, 1, 2))
        mk = dict(num_layers=L, hidden_size=rng.choice((64, 128, 256)), seq_len=rng.choice((32, 64)),
                  t_forward=rng.choice((1.0, 1.5)), t_input_grad=rng.choice((1.0, 2.0)),
                  t_weight_grad=rng.choice((1.0, 0.5)), t_optstep=rng.choice((0.0, 0.25)))
        pk = dict(pp_size=P, dp_size=rng.choice((1, 2, 4)), microbatches=B, unit_size=U, stages_per_device=V,
                  microbatch_samples=rng.choice((1, 2)), inter_node_dp=n,
                  hybrid_mode=rng.choice(("dp_outer", "zero1_outer")),
                  recompute=rng.choice(("none", "full")) if V > 1 else "none")
        ck = {"intra_node_bandwidth": rng.choice((1e5, 1e6, 1e30)), "inter_node_bandwidth": rng.choice((1e4, 1e5)),
              "per_collective_latency": rng.choice((0.0, 0.125)), "overlap_with_compute": rng.random() < 0.8}
        cases.append(record(f"rand{i}", mk, pk, ck, render=(P * B <= 24)))
    OUT.write_text(json.dumps(cases, indent=1, sort_keys=True) + "\n")
    print(f"wrote {len(cases)} cases to {OUT}")


if __name__ == "__main__":
    main()
