"""Generate the closed-form cost-model fixtures from the REAL reference package.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_costmodel_golden.py

Writes ``tests/golden/costmodel.json``: for the five BASELINE configs, the reference's own
test configs (pkg/tests/test_costmodel.py) and 300 seeded random configs, the ``repr`` of
every closed form (`costmodel.py:65-189`): tp / zeropp traffic, crossover, bubble formula,
memory formula, every table2_row (or its ConfigError text) and figure1_curve.
"""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import zeroppsim as R  # noqa: E402

OUT = Path(__file__).with_name("costmodel.json")


def _try(fn):
    try:
        return repr(fn())
    except R.ConfigError as e:
        return f"ConfigError: {e}"


def record(model_kw: dict, par_kw: dict) -> dict:
    m = R.ModelSpec(**model_kw)
    c = R.ParallelConfig(**par_kw)
    rows = {}
    for meth in R.Method:
        rows[meth.value] = _try(lambda: (lambda r: (r.method.value, r.bubble_ratio, r.weight_mem, r.activation_mem,
                                                    r.comm_volume_per_block, r.crossover_satisfied))(
            R.table2_row(meth, m, c)))
    return {"model": model_kw, "parallel": par_kw,
            "tp": repr(R.tp_comm_volume(m, c)), "zeropp": repr(R.zeropp_comm_volume(m, c)),
            "crossover": R.crossover(m, c), "bubble": repr(R.bubble_formula(c)),
            "memory": repr(R.memory_formula(m, c)), "rows": rows,
            "figure1": _try(lambda: R.figure1_curve(m, [1, 2, 8, 64, 512]))}


def main() -> None:
    cases = []
    base = [
        ({"num_layers": 4, "hidden_size": 256, "seq_len": 128}, dict(pp_size=2, dp_size=2, microbatches=8, unit_size=4, stages_per_device=2)),
        ({"num_layers": 24, "hidden_size": 2048, "seq_len": 2048}, dict(pp_size=2, dp_size=4, microbatches=16, unit_size=8, stages_per_device=2)),
        ({"num_layers": 32, "hidden_size": 4096, "seq_len": 2048}, dict(pp_size=2, dp_size=4, microbatches=16, unit_size=8, stages_per_device=2)),
        ({"num_layers": 32, "hidden_size": 4096, "seq_len": 4096}, dict(pp_size=4, dp_size=2, microbatches=32, unit_size=8, stages_per_device=2)),
        ({"num_layers": 40, "hidden_size": 5120, "seq_len": 2048}, dict(pp_size=8, dp_size=1, microbatches=128, unit_size=16, stages_per_device=1)),
        # pkg/tests/test_costmodel.py configs
        ({"num_layers": 48, "hidden_size": 5120, "seq_len": 1024, "bytes_per_element": 1},
         dict(pp_size=4, dp_size=8, microbatches=16, unit_size=16, stages_per_device=1, microbatch_samples=4)),
        ({"num_layers": 48, "hidden_size": 8, "seq_len": 8, "weight_mem_per_layer": 1.0,
          "act_mem_per_layer_per_microbatch": 1.0}, dict(pp_size=4, dp_size=8, microbatches=12, unit_size=6, stages_per_device=2)),
    ]
    for m, p in base:
        cases.append(record(m, p))
    rng = random.Random(20240817)
    while len(cases) < 307:
        P, V = rng.choice([1, 2, 3, 4, 8]), rng.choice([1, 2, 3, 4, 5])
        U = rng.randint(1, 12)
        B = U * rng.randint(1, 6)
        L = P * V * rng.randint(1, 4)
        m = {"num_layers": L, "hidden_size": rng.choice([64, 256, 1024, 4096, 5120]),
             "seq_len": rng.choice([128, 1024, 2048, 4096]), "bytes_per_element": rng.choice([1, 2, 4])}
        if rng.random() < 0.3:
            m["weight_mem_per_layer"] = rng.choice([1.0, 3.5, 1e9])
            m["act_mem_per_layer_per_microbatch"] = rng.choice([1.0, 0.25, 7e8])
        p = dict(pp_size=P, dp_size=rng.choice([1, 2, 4, 8]), microbatches=B, unit_size=U, stages_per_device=V,
                 microbatch_samples=rng.choice([1, 2, 4]))
        try:
            cases.append(record(m, p))
        except R.ConfigError:
            continue
    errors = {"figure1_empty": _try(lambda: R.figure1_curve(R.ModelSpec(num_layers=4, hidden_size=64, seq_len=64), [])),
              "figure1_zero": _try(lambda: R.figure1_curve(R.ModelSpec(num_layers=4, hidden_size=64, seq_len=64), [0]))}
    OUT.write_text(json.dumps({"cases": cases, "errors": errors,
                               "table_methods": [m.value for m in R.TABLE_METHODS]}, sort_keys=True))
    print(f"wrote {OUT} ({len(cases)} cases)")


if __name__ == "__main__":
    main()
