"""Generate the schedule golden fixtures from the REAL reference package.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes ``tests/golden/schedules.json``: for every case the config, per-device
sha256 of ``task_id:cost!r:bytes!r`` (so ids, float costs and float bytes are
pinned bit-for-bit), sha256 of the sorted edge list, task/edge counts and the
validator's verdict; small cases also carry the full per-device id lists.
Cases: the five BASELINE configs, the reference's own
golden/test configs (pkg/tests/test_schedules.py:27-205), 400 seeded random
configs (P up to 8, V up to 5, recompute, both outer modes, non-uniform
costs), and the reference ``fuzz_check`` summaries (validation.py:319-340).
"""

from __future__ import annotations

import hashlib
import json
import random
import sys
import warnings
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import zeroppsim as R  # noqa: E402

OUT = Path(__file__).with_name("schedules.json")


def _h(s: str) -> str:
    return hashlib.sha256(s.encode()).hexdigest()[:32]


def record(name: str, model_kw: dict, par_kw: dict, full: bool) -> dict:
    m = R.ModelSpec(**model_kw)
    pk = dict(par_kw)
    pk["hybrid_mode"] = R.HybridMode(pk.get("hybrid_mode", "dp_outer"))
    pk["recompute"] = R.RecomputeMode(pk.get("recompute", "none"))
    c = R.ParallelConfig(**pk)
    pl = R.make_placement(c, m)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        s = R.generate(m, c, pl)
    dev_payload = [" ".join(f"{t.task_id}:{t.cost!r}:{t.bytes!r}" for t in lst)
                   for lst in s.per_device]
    edges = sorted((a.task_id, b.task_id) for a, b in s.edges)
    rec = {
        "name": name,
        "model": model_kw,
        "parallel": par_kw,
        "tasks": s.task_count(),
        "edges": len(edges),
        "device_sha": [_h(x) for x in dev_payload],
        "edges_sha": _h("\n".join(f"{a} {b}" for a, b in edges)),
        "violations": [str(v) for v in R.validate(s, pl, c)],
    }
    if full:
        rec["per_device"] = [[f"{t.task_id}:{t.cost!r}:{t.bytes!r}" for t in lst]
                             for lst in s.per_device]
    return rec


def main() -> None:
    cases = []
    base = [
        ("C1_tiny", dict(num_layers=4, hidden_size=256, seq_len=128),
         dict(pp_size=2, dp_size=2, microbatches=8, unit_size=4, stages_per_device=2), True),
        ("C2_gpt1p3b", dict(num_layers=24, hidden_size=2048, seq_len=2048),
         dict(pp_size=2, dp_size=4, microbatches=16, unit_size=8, stages_per_device=2), False),
        ("C3_gpt6p2b", dict(num_layers=32, hidden_size=4096, seq_len=2048),
         dict(pp_size=2, dp_size=4, microbatches=16, unit_size=8, stages_per_device=2), False),
        ("C4_llama7b", dict(num_layers=32, hidden_size=4096, seq_len=4096),
         dict(pp_size=4, dp_size=2, microbatches=32, unit_size=8, stages_per_device=2), False),
        ("C5_gpt13b", dict(num_layers=40, hidden_size=5120, seq_len=2048),
         dict(pp_size=8, dp_size=1, microbatches=128, unit_size=16, stages_per_device=1), False),
        ("bench_6p2b_1x1", dict(num_layers=32, hidden_size=4096, seq_len=2048),
         dict(pp_size=1, dp_size=1, microbatches=16, unit_size=4, stages_per_device=1), True),
    ]
    for b in (8, 32, 64):
        base.append((f"C3_gpt6p2b_B{b}", dict(num_layers=32, hidden_size=4096, seq_len=2048),
                     dict(pp_size=2, dp_size=4, microbatches=b, unit_size=8,
                          stages_per_device=2), False))
    # the reference's own test configs (pkg/tests/conftest.py:12-22 abstract units)
    abstract = dict(hidden_size=64, seq_len=16, weight_mem_per_layer=1.0,
                    act_mem_per_layer_per_microbatch=1.0)
    ref_tests = [
        ("ref_golden_two_device", 2, dict(pp_size=2, dp_size=2, microbatches=2, unit_size=1)),
        ("ref_counts_a", 2, dict(pp_size=2, dp_size=2, microbatches=4, unit_size=2)),
        ("ref_counts_b", 4, dict(pp_size=2, dp_size=2, microbatches=4, unit_size=4,
                                 stages_per_device=2)),
        ("ref_counts_c", 8, dict(pp_size=4, dp_size=2, microbatches=12, unit_size=3,
                                 stages_per_device=2)),
        ("ref_counts_d", 6, dict(pp_size=3, dp_size=2, microbatches=6, unit_size=2,
                                 stages_per_device=2)),
        ("ref_breadth_first", 8, dict(pp_size=4, dp_size=2, microbatches=4, unit_size=4,
                                      stages_per_device=2)),
        ("ref_recompute", 8, dict(pp_size=4, dp_size=2, microbatches=4, unit_size=4,
                                  stages_per_device=2, recompute="full")),
        ("ref_validation_base", 8, dict(pp_size=4, dp_size=2, microbatches=8, unit_size=4,
                                        stages_per_device=2, inter_node_dp=2)),
    ]
    for name, L, pk in ref_tests:
        base.append((name, dict(num_layers=L, **abstract), pk, True))
    base.append(("ref_costs", dict(num_layers=12, t_forward=1.0, t_input_grad=0.5,
                                   t_weight_grad=0.25, t_optstep=0.125, **abstract),
                 dict(pp_size=2, dp_size=2, microbatches=2, unit_size=2, stages_per_device=3),
                 True))
    for name, mk, pk, full in base:
        cases.append(record(name, mk, pk, full))

    rng = random.Random(20240817)
    cost_sets = [(1.0, 1.0, 1.0, 0.0), (1.0, 2.0, 1.0, 0.5), (1.3, 0.7, 0.9, 0.1),
                 (1.0, 1.0, 0.5, 0.0), (2.0, 1.0, 3.0, 0.25)]
    for i in range(400):
        P = rng.choice((1, 2, 3, 4, 6, 8))
        V = rng.randint(1, 5)
        U = rng.randint(1, 8)
        B = U * rng.randint(1, max(1, 48 // U))
        tf, ti, tw, to = rng.choice(cost_sets)
        mk = dict(num_layers=P * V * rng.choice((1, 2, 3)), hidden_size=rng.choice((64, 4096)),
                  seq_len=rng.choice((16, 2048)), t_forward=tf, t_input_grad=ti,
                  t_weight_grad=tw, t_optstep=to)
        pk = dict(pp_size=P, dp_size=rng.choice((1, 2, 4, 8)), microbatches=B, unit_size=U,
                  stages_per_device=V, inter_node_dp=rng.choice((1, 2, 4)),
                  hybrid_mode=rng.choice(("dp_outer", "zero1_outer")),
                  recompute=rng.choice(("none", "none", "full")))
        cases.append(record(f"fuzz_{i}", mk, pk, False))

    fuzz = []
    for seed, trials in ((7, 60), (20240817, 100)):
        s = R.fuzz_check(seed, trials)
        fuzz.append({"seed": seed, "trials": trials, "ok": s.ok,
                     "generated_clean": s.generated_clean,
                     "mutations_caught": s.mutations_caught})
    OUT.write_text(json.dumps({"generator": "zeroppsim (reference) generate/validate",
                               "cases": cases, "fuzz_check": fuzz}, indent=1))
    print(f"wrote {OUT} with {len(cases)} cases")


if __name__ == "__main__":
    main()
