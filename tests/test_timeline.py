"""Measured-timeline adapter (CPU part): calibrate() recovers the costs of a known
timeline and predict() reproduces it; summarize() matches simulate() on the same times."""

import dataclasses

import pytest

import paper_2402_03791_b200 as Z
from paper_2402_03791_b200.engine.timeline import calibrate, model_flops_per_token, predict
from paper_2402_03791_b200.simulation import simulate, summarize


def _setup(recompute="none"):
    m = Z.ModelSpec(num_layers=8, hidden_size=256, seq_len=128)
    c = Z.ParallelConfig(pp_size=2, dp_size=2, microbatches=8, unit_size=4, stages_per_device=2,
                         recompute=Z.RecomputeMode(recompute))
    pl = Z.make_placement(c, m)
    return m, c, pl, Z.generate(m, c, pl)


@pytest.mark.parametrize("recompute", ["none", "full"])
def test_calibrate_recovers_costs_and_predict_reproduces(recompute):
    m, c, pl, s = _setup(recompute)
    # a "measured" timeline: the executed order with known per-layer costs (ms) and bandwidth
    truth = dataclasses.replace(m, t_forward=1.5, t_input_grad=2.25, t_weight_grad=1.25, t_optstep=0.5)
    costs = Z.CommCostModel(intra_node_bandwidth=4.0e5, inter_node_bandwidth=4.0e5)
    measured = predict(s, truth, costs, c, pl)
    fitted, fcosts = calibrate(measured, s, m, pl)
    assert (fitted.t_forward, fitted.t_input_grad, fitted.t_weight_grad) == (1.5, 2.25, 1.25)
    assert fitted.t_optstep == pytest.approx(0.5)
    assert fcosts.intra_node_bandwidth == pytest.approx(4.0e5)
    again = predict(s, fitted, fcosts, c, pl)
    assert again.makespan == pytest.approx(measured.makespan)
    assert again.bubble_ratios == pytest.approx(measured.bubble_ratios)
    # the executed ORDER is kept (not regenerated with the new costs)
    assert [[t.task_id for t in lst] for lst in s.per_device] == \
        [[t.task_id for t in lst] for lst in s.per_device]


def test_summarize_equals_simulate_on_same_times():
    m, c, pl, s = _setup()
    costs = Z.CommCostModel(intra_node_bandwidth=1e6, inter_node_bandwidth=1e6, per_collective_latency=0.1)
    r = simulate(s, m, c, pl, costs)
    r2 = summarize(s, m, c, pl, r.task_times, {"loss": 1.0})
    assert (r2.makespan, r2.per_device_busy, r2.peak_mem, r2.mem_trace) == \
        (r.makespan, r.per_device_busy, r.peak_mem, r.mem_trace)
    assert r2.extras["loss"] == 1.0


def test_model_flops_gpt_6p2b():
    from paper_2402_03791_b200.engine import GPTSpec
    assert model_flops_per_token(GPTSpec.gpt_6p2b()) / 1e9 == pytest.approx(43.11, abs=0.01)


def test_engine_tokens_equal_oracle_tokens():
    from oracle.gpt_oracle import make_tokens
    from paper_2402_03791_b200.engine.data import synthetic_tokens
    import torch
    assert torch.equal(synthetic_tokens(2, 2, 3, 1, 16, 50304), make_tokens(2, 2, 3, 1, 16, 50304))
