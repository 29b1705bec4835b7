"""Generator properties (mirrors the reference's pkg/tests/test_schedules.py)."""

import warnings

import pytest

from conftest import mk_cfg, mk_model
from paper_2402_03791_b200 import (
    ConfigError, RecomputeMode, ScheduleVariant, TaskKind, apply_recompute, expected_edges,
    generate, make_placement,
)


def build(m, cfg, variant=ScheduleVariant.ZEROPP):
    pl = make_placement(cfg, m)
    return generate(m, cfg, pl, variant), pl


def test_golden_two_device_single_unit():
    # test_schedules.py:27-42
    sched, _ = build(mk_model(layers=2), mk_cfg(P=2, D=2, B=2, U=1))
    for d in range(2):
        want = []
        for u in range(2):
            want += [f"AG_PARAM.d{d}.s{d}.u{u}.fwd", f"F.d{d}.s{d}.m{u}.u{u}",
                     f"AG_PARAM.d{d}.s{d}.u{u}.bwd", f"B.d{d}.s{d}.m{u}.u{u}",
                     f"W.d{d}.s{d}.m{u}.u{u}", f"RS_GRAD.d{d}.s{d}.u{u}"]
        want.append(f"OPT.d{d}")
        assert [t.task_id for t in sched.per_device[d]] == want


@pytest.mark.parametrize("P,V,U,B", [(2, 1, 2, 4), (2, 2, 4, 4), (4, 2, 3, 12), (3, 2, 2, 6)])
def test_task_counts(P, V, U, B):
    sched, _ = build(mk_model(layers=P * V), mk_cfg(P=P, D=2, B=B, U=U, V=V))
    for lst in sched.per_device:
        kinds = [t.kind for t in lst]
        for k in (TaskKind.F, TaskKind.B, TaskKind.W):
            assert kinds.count(k) == B * V
        assert kinds.count(TaskKind.AG_PARAM) == 2 * V * (B // U)
        assert kinds.count(TaskKind.RS_GRAD) == V * (B // U)
        assert kinds.count(TaskKind.OPT) == 1


def test_units_do_not_interleave():
    sched, _ = build(mk_model(layers=8), mk_cfg(P=4, D=2, B=12, U=3, V=2))
    for lst in sched.per_device:
        units = [t.unit for t in lst if t.is_compute and t.unit is not None]
        assert units == sorted(units)


def test_w_follows_its_b_on_the_same_device():
    # the engine relies on it: W(s,m) re-uses the dY stash B(s,m) produced
    for P, V, U, B in [(2, 2, 4, 8), (4, 2, 8, 16), (3, 3, 2, 6), (1, 1, 4, 8)]:
        sched, _ = build(mk_model(layers=P * V), mk_cfg(P=P, D=2, B=B, U=U, V=V))
        for lst in sched.per_device:
            pos = {(t.kind, t.stage, t.microbatch): i for i, t in enumerate(lst)}
            for (k, s, m), i in pos.items():
                if k is TaskKind.W:
                    assert pos[(TaskKind.B, s, m)] < i


def test_recompute_inserts_r_before_early_round_backward():
    m = mk_model(layers=8)
    sched, _ = build(m, mk_cfg(P=4, D=2, B=4, U=4, V=2, recompute=RecomputeMode.FULL))
    for lst in sched.per_device:
        comp = [t for t in lst if t.is_compute]
        rs = [i for i, t in enumerate(comp) if t.kind is TaskKind.R]
        assert len(rs) == 4
        for i in rs:
            nxt = comp[i + 1]
            assert nxt.kind is TaskKind.B and nxt.stage == comp[i].stage
            assert nxt.microbatch == comp[i].microbatch and comp[i].stage // 4 == 0


def test_recompute_single_stage_warns_and_is_noop():
    m = mk_model(layers=4)
    cfg = mk_cfg(P=4, D=2, B=4, U=4, V=1)
    pl = make_placement(cfg, m)
    base = generate(m, cfg, pl)
    with pytest.warns(UserWarning, match="no effect"):
        same = apply_recompute(base, m, cfg, pl)
    assert same.per_device == base.per_device


def test_recompute_rejected_for_bfpp():
    with pytest.raises(ConfigError, match="recompute"):
        build(mk_model(layers=4), mk_cfg(P=2, D=1, B=4, U=4, recompute=RecomputeMode.FULL),
              ScheduleVariant.BFPP)


def test_edges_match_expected_edges():
    m = mk_model(layers=8)
    for variant, U in ((ScheduleVariant.ZEROPP, 2), (ScheduleVariant.BFPP, 4)):
        cfg = mk_cfg(P=2, D=2, B=4, U=U, V=2)
        pl = make_placement(cfg, m)
        assert generate(m, cfg, pl, variant).edges == expected_edges(variant, pl, cfg)


def test_costs_follow_layer_counts():
    m = mk_model(layers=12, t_forward=1.0, t_input_grad=0.5, t_weight_grad=0.25, t_optstep=0.125)
    sched, _ = build(m, mk_cfg(P=2, D=2, B=2, U=2, V=3))
    want = {TaskKind.F: 2.0, TaskKind.B: 1.0, TaskKind.W: 0.5, TaskKind.OPT: 0.75}
    for t in sched.tasks():
        if t.kind in want:
            assert t.cost == want[t.kind]


def test_classic_baselines_are_out_of_scope():
    from paper_2402_03791_b200 import ConfigError
    with pytest.raises(ConfigError, match="outside the engine's hot path"):
        build(mk_model(layers=4), mk_cfg(P=4, D=1, B=8, U=8), ScheduleVariant.GPIPE)
