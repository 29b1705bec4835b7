"""Validator mutation tests (mirrors the reference's pkg/tests/test_validation.py)."""

import dataclasses

import pytest

from conftest import mk_cfg, mk_model
from paper_2402_03791_b200 import (
    Schedule, TaskKind, ViolationKind, fuzz_check, generate, make_placement, validate,
)


@pytest.fixture
def base():
    m = mk_model(layers=8)
    cfg = mk_cfg(P=4, D=2, B=8, U=4, V=2, inter_node_dp=2)
    pl = make_placement(cfg, m)
    return cfg, pl, generate(m, cfg, pl)


def mutate(sched, d, fn):
    per_device = [list(x) for x in sched.per_device]
    fn(per_device[d])
    return Schedule(sched.variant, per_device, sched.edges)


def kinds_of(sched, pl, cfg):
    return {v.kind for v in validate(sched, pl, cfg)}


def test_clean(base):
    cfg, pl, s = base
    assert validate(s, pl, cfg) == []


def test_b_before_f_flagged(base):
    cfg, pl, s = base
    last = cfg.num_stages - 1

    def fn(lst):
        b = lst.pop(next(i for i, t in enumerate(lst) if t.kind is TaskKind.B
                         and t.stage == last and t.microbatch == 0))
        lst.insert(next(i for i, t in enumerate(lst) if t.kind is TaskKind.F
                        and t.stage == last and t.microbatch == 0), b)
    assert ViolationKind.DEP_ORDER in kinds_of(mutate(s, cfg.pp_size - 1, fn), pl, cfg)


def test_missing_duplicate_wrongdevice(base):
    cfg, pl, s = base
    miss = mutate(s, 2, lambda l: l.remove(next(t for t in l if t.kind is TaskKind.W)))
    assert ViolationKind.MISSING_TASK in kinds_of(miss, pl, cfg)
    dup = mutate(s, 0, lambda l: l.append(next(t for t in l if t.kind is TaskKind.F)))
    assert ViolationKind.DUPLICATE_TASK in kinds_of(dup, pl, cfg)

    def move(l):
        l[1] = dataclasses.replace(l[1], device=(l[1].device + 1) % cfg.pp_size)
    assert ViolationKind.DEVICE_MISMATCH in kinds_of(mutate(s, 0, move), pl, cfg)


def test_unit_leak(base):
    cfg, pl, s = base

    def fn(l):
        t = l.pop(next(i for i, t in enumerate(l) if t.is_compute and t.unit == 1))
        l.insert(next(i for i, x in enumerate(l) if x.is_compute and x.unit == 0
                      and x.kind in (TaskKind.B, TaskKind.W)), t)
    assert ViolationKind.UNIT_LEAK in kinds_of(mutate(s, 0, fn), pl, cfg)


def test_gather_after_use_and_opt_first(base):
    cfg, pl, s = base

    def late(l):
        ag = l.pop(next(i for i, t in enumerate(l)
                        if t.kind is TaskKind.AG_PARAM and t.phase == "fwd"))
        j = next(j for j, t in enumerate(l)
                 if t.kind is TaskKind.F and t.stage == ag.stage and t.unit == ag.unit)
        l.insert(j + 1, ag)
    assert ViolationKind.DEP_ORDER in kinds_of(mutate(s, 3, late), pl, cfg)

    def hoist(l):
        l.insert(0, l.pop(next(i for i, t in enumerate(l) if t.kind is TaskKind.OPT)))
    assert validate(mutate(s, 0, hoist), pl, cfg) != []


def test_fuzz():
    s = fuzz_check(seed=7, trials=60)
    assert s.ok, s.failures[:5]
