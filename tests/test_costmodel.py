"""Closed-form cost model (`costmodel.py`): bit-exact against fixtures generated from the real
reference (tests/golden/make_costmodel_golden.py), plus the reference's own known answers
(pkg/tests/test_costmodel.py)."""

import json
from pathlib import Path

import pytest

from paper_2402_03791_b200 import (TABLE_METHODS, ConfigError, Method, ModelSpec, ParallelConfig, bubble_formula,
                                   crossover, figure1_curve, memory_formula, table2_row, tp_comm_volume,
                                   zeropp_comm_volume)

GOLD = json.loads((Path(__file__).parent / "golden" / "costmodel.json").read_text())


def _try(fn):
    try:
        return repr(fn())
    except ConfigError as e:
        return f"ConfigError: {e}"


@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: f"L{c['model']['num_layers']}h{c['model']['hidden_size']}"
                         f"P{c['parallel']['pp_size']}U{c['parallel']['unit_size']}")
def test_closed_forms_match_reference(case):
    m, c = ModelSpec(**case["model"]), ParallelConfig(**case["parallel"])
    assert repr(tp_comm_volume(m, c)) == case["tp"]
    assert repr(zeropp_comm_volume(m, c)) == case["zeropp"]
    assert crossover(m, c) == case["crossover"]
    assert repr(bubble_formula(c)) == case["bubble"]
    assert repr(memory_formula(m, c)) == case["memory"]
    for meth in Method:
        got = _try(lambda: (lambda r: (r.method.value, r.bubble_ratio, r.weight_mem, r.activation_mem,
                                       r.comm_volume_per_block, r.crossover_satisfied))(table2_row(meth, m, c)))
        assert got == case["rows"][meth.value], meth
    assert _try(lambda: figure1_curve(m, [1, 2, 8, 64, 512])) == case["figure1"]


def test_errors_and_table_methods():
    m = ModelSpec(num_layers=4, hidden_size=64, seq_len=64)
    assert _try(lambda: figure1_curve(m, [])) == GOLD["errors"]["figure1_empty"]
    assert _try(lambda: figure1_curve(m, [0])) == GOLD["errors"]["figure1_zero"]
    assert [x.value for x in TABLE_METHODS] == GOLD["table_methods"]


H5120 = ModelSpec(num_layers=48, hidden_size=5120, seq_len=1024, bytes_per_element=1)
ABSTRACT = ModelSpec(num_layers=48, hidden_size=8, seq_len=8, weight_mem_per_layer=1.0,
                     act_mem_per_layer_per_microbatch=1.0)


def cfg(P=4, D=8, B=16, U=16, V=1, b=1):
    return ParallelConfig(pp_size=P, dp_size=D, microbatches=B, unit_size=U, stages_per_device=V,
                          microbatch_samples=b)


def test_reference_known_answers():
    assert tp_comm_volume(H5120, cfg(B=16, U=16, b=4)) == 2_684_354_560
    assert zeropp_comm_volume(H5120, cfg(B=16, U=16)) == 943_718_400
    assert zeropp_comm_volume(H5120, cfg(B=16, U=8)) == 2 * 943_718_400
    assert min(u for u in range(1, 17) if crossover(H5120, cfg(B=4 * u, U=u, b=2))) == 12
    assert bubble_formula(cfg(P=4, B=8, U=4)) == 6.0
    assert bubble_formula(cfg(P=4, B=14, U=7)) == 0.0
    assert memory_formula(ABSTRACT, cfg(B=12, U=6, V=2)) == (7.5, 72.0)
    row = table2_row(Method.ZEROPP, ABSTRACT, cfg(B=8, U=8, V=2))
    assert row.bubble_ratio == 0.0 and row.activation_mem == 1.75 * 48 and row.weight_mem == 7.5
    with pytest.raises(ConfigError, match="gpipe assumes"):
        table2_row(Method.GPIPE, ABSTRACT, cfg(V=2))
    with pytest.raises(ConfigError, match="no closed-form"):
        table2_row(Method.BFPP, ABSTRACT, cfg())
