"""Config API parity (mirrors pkg/tests/test_config.py)."""

import json

import pytest

from paper_2402_03791_b200 import (
    ConfigError, HybridMode, ModelSpec, ParallelConfig, load_config, make_placement,
)


def test_defaults():
    m = ModelSpec(num_layers=32, hidden_size=4096, seq_len=2048)
    assert m.weight_mem_per_layer == 12 * 4096**2 * 2
    assert m.act_mem(1) == 2048 * 4096 * 2 * 34.0 and m.act_mem(2) == 2 * m.act_mem(1)


@pytest.mark.parametrize("kw", [dict(num_layers=0), dict(t_forward=-1.0),
                                dict(weight_mem_per_layer=0.0), dict(activation_constant=0)])
def test_model_rejects(kw):
    base = dict(num_layers=4, hidden_size=8, seq_len=8)
    base.update(kw)
    with pytest.raises(ConfigError):
        ModelSpec(**base)


def test_parallel_rejects():
    with pytest.raises(ConfigError, match="B mod U"):
        ParallelConfig(pp_size=2, dp_size=1, microbatches=6, unit_size=4)
    with pytest.raises(ConfigError, match="unit_size"):
        ParallelConfig(pp_size=2, dp_size=1, microbatches=2, unit_size=4)


def test_placement_loops():
    cfg = ParallelConfig(pp_size=2, dp_size=4, microbatches=16, unit_size=8, stages_per_device=2)
    pl = make_placement(cfg, ModelSpec(num_layers=32, hidden_size=64, seq_len=8))
    assert pl.stage_to_device == (0, 1, 0, 1)
    assert pl.stage_to_layers == ((0, 8), (8, 16), (16, 24), (24, 32))
    assert pl.device_stages(1) == (1, 3)
    with pytest.raises(ConfigError, match="L mod"):
        make_placement(cfg, ModelSpec(num_layers=6, hidden_size=64, seq_len=8))


def test_load_config(tmp_path):
    p = tmp_path / "c.json"
    p.write_text(json.dumps({
        "model": {"num_layers": 8, "hidden_size": 512, "seq_len": 128},
        "parallel": {"pp_size": 2, "dp_size": 2, "microbatches": 8, "unit_size": 4,
                     "stages_per_device": 2, "hybrid_mode": "zero1_outer"},
        "costs": {"intra_node_bandwidth": "inf", "inter_node_bandwidth": 5e9}}))
    m, c, k = load_config(p)
    assert c.hybrid_mode is HybridMode.ZERO1_OUTER and k.intra_node_bandwidth == float("inf")
    raw = json.loads(p.read_text())
    raw["model"]["bogus"] = 1
    p.write_text(json.dumps(raw))
    with pytest.raises(ConfigError, match="unknown key"):
        load_config(p)
