"""Executed NCCL bytes vs the reference's byte model.

``nccl_bytes_per_step`` is what the executor hands to NCCL (the GPU tests check the running
engine reports exactly this, per rank).  Here it is tied to the reference's accounting:

* per AG_PARAM / RS_GRAD task the reference charges ``((D-1)/D) * M_w * layers``
  (`schedules.py:72-78`, M_w = 12 h^2 bytes-per-element); the engine moves its real flat stage,
  i.e. that plus ``((D-1)/D) * 2 B * extra`` where extra = biases, LayerNorm parameters,
  embeddings / LM head and alignment padding of the stage -- checked task by task through the
  simulator's ``comm_bytes_intra`` (pinned to the reference in test_simulation_golden.py);
* the per-block part equals the closed form ``(D-1)/D * zeropp_comm_volume`` per layer
  (`costmodel.py:82-95`), and the inter-node tail matches ``comm_bytes_inter``.
"""

import pytest

from paper_2402_03791_b200 import (CommCostModel, HybridMode, ModelSpec, ParallelConfig, generate, make_placement, simulate,
                                   zeropp_comm_volume)
from paper_2402_03791_b200.engine import GPTSpec
from paper_2402_03791_b200.engine.model import nccl_bytes_per_step, optimizer_sub, stage_layout

COSTS = CommCostModel(intra_node_bandwidth=900e9, inter_node_bandwidth=50e9)
CASES = [  # (spec, P, D, B, U, V, n, mode)
    (GPTSpec.tiny(), 2, 2, 8, 4, 2, 1, "dp_outer"),                         # C1
    (GPTSpec.gpt_1p3b(), 2, 4, 16, 8, 2, 1, "dp_outer"),                    # C2
    (GPTSpec.gpt_6p2b(), 2, 4, 16, 8, 2, 1, "dp_outer"),                    # C3
    (GPTSpec.llama_7b(), 4, 2, 32, 8, 2, 1, "dp_outer"),                    # C4
    (GPTSpec(num_layers=40, hidden=5120, heads=40, seq_len=2048), 8, 1, 128, 16, 1, 1, "dp_outer"),  # C5
    (GPTSpec.gpt_6p2b(), 1, 4, 8, 2, 2, 1, "dp_outer"),
    (GPTSpec.tiny(), 2, 2, 8, 4, 2, 2, "dp_outer"),
    (GPTSpec.tiny(), 2, 2, 8, 4, 1, 2, "zero1_outer"),
    (GPTSpec.tiny(), 1, 2, 4, 2, 2, 4, "zero1_outer"),
]


def _setup(spec, P, D, B, U, V, n, mode):
    per_layer = 12 * spec.hidden ** 2
    model = ModelSpec(num_layers=spec.num_layers, hidden_size=spec.hidden, seq_len=spec.seq_len,
                      weight_mem_per_layer=float(2 * per_layer))
    cfg = ParallelConfig(pp_size=P, dp_size=D, microbatches=B, unit_size=U, stages_per_device=V,
                         inter_node_dp=n, hybrid_mode=HybridMode(mode))
    pl = make_placement(cfg, model)
    return model, cfg, pl, generate(model, cfg, pl), per_layer


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"L{c[0].num_layers}h{c[0].hidden}P{c[1]}D{c[2]}n{c[6]}{c[7]}")
def test_executed_bytes_equal_reference_model_plus_real_stage_extras(case):
    spec, P, D, B, U, V, n, mode = case
    model, cfg, pl, sched, per_layer = _setup(*case)
    sim = simulate(sched, model, cfg, pl, COSTS)
    sub = optimizer_sub(cfg)
    total_intra = total_inter = 0
    for p in range(P):
        intra, inter = nccl_bytes_per_step(spec, cfg, pl, sched, p)
        total_intra += intra
        total_inter += inter
        # task by task: reference bytes + the stage's extra parameters
        expect = 0.0
        for t in sched.per_device[p]:
            if t.kind.value in ("AG_PARAM", "RS_GRAD"):
                lay = stage_layout(spec, t.stage, cfg.num_stages, pl.stage_to_layers[t.stage], D, sub)
                layers = pl.stage_to_layers[t.stage][1] - pl.stage_to_layers[t.stage][0]
                extra = lay.numel - per_layer * layers
                assert extra >= 0
                expect += t.bytes + (D - 1) / D * 2 * extra
        assert intra == pytest.approx(expect, rel=1e-12, abs=1e-6)
        # per-block closed form: 3 movements of 12 h^2 per unit, (D-1)/D on a ring
        block_part = sum(t.bytes for t in sched.per_device[p] if t.kind.value in ("AG_PARAM", "RS_GRAD"))
        layers_p = sum(pl.stage_to_layers[s][1] - pl.stage_to_layers[s][0] for s in pl.device_stages(p))
        assert block_part == pytest.approx((D - 1) / D * zeropp_comm_volume(model, cfg) * layers_p, rel=1e-12)
    extras_total = sum(
        (D - 1) / D * 2 * (stage_layout(spec, t.stage, cfg.num_stages, pl.stage_to_layers[t.stage], D, sub).numel
                           - per_layer * (pl.stage_to_layers[t.stage][1] - pl.stage_to_layers[t.stage][0]))
        for p in range(P) for t in sched.per_device[p] if t.kind.value in ("AG_PARAM", "RS_GRAD"))
    assert total_intra == pytest.approx(sim.comm_bytes_intra + extras_total, rel=1e-12, abs=1e-6)
    if n == 1:
        assert total_inter == 0 and sim.comm_bytes_inter == 0
    else:
        assert total_inter > 0 and sim.comm_bytes_inter > 0


def test_single_gpu_moves_nothing():
    spec = GPTSpec.gpt_6p2b()
    model, cfg, pl, sched, _ = _setup(spec, 1, 1, 8, 2, 1, 1, "dp_outer")
    assert nccl_bytes_per_step(spec, cfg, pl, sched, 0) == (0, 0)
    assert simulate(sched, model, cfg, pl, COSTS).comm_bytes_intra == 0
