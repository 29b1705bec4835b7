"""The parity harness itself (CPU): per-tensor gradient checks catch a single wrong small
tensor that the whole-stage cosine would miss (a zeroed bias gradient, an inverted
LayerNorm beta gradient)."""

import types

import torch

from engine_harness import build, compare_shards, flat_stage, oracle_for
from oracle.gpt_oracle import make_tokens
from paper_2402_03791_b200.engine import GPTSpec
from paper_2402_03791_b200.engine.model import stage_layout


def _fake_runtime(spec, cfg, pl, grads_o, new_o):
    """A P x D = 1 x 1 'runtime' whose shards are exactly the oracle's."""
    stages, captured = {}, {}
    for s in range(cfg.num_stages):
        lay = stage_layout(spec, s, cfg.num_stages, pl.stage_to_layers[s], 1)
        master = flat_stage(spec, cfg, pl, s, new_o)
        bf = master.to(torch.bfloat16)
        stages[s] = types.SimpleNamespace(lay=lay, nsub=lay.numel, sub=1, master=master, sub_bf16=bf,
                                          shard_bf16=bf)
        captured[s] = flat_stage(spec, cfg, pl, s, grads_o)
    return types.SimpleNamespace(stages=stages, captured=captured, z=0, node=0)


def _setup():
    spec = GPTSpec.tiny()
    model, cfg, pl, sched = build(spec, 1, 1, 2, 1, 2)
    tokens = make_tokens(1, 1, 2, 1, spec.seq_len, spec.vocab)
    _, grads_o, new_o = oracle_for(spec, cfg, pl, tokens[0])
    return spec, cfg, pl, grads_o, new_o


def test_harness_accepts_oracle_and_rejects_one_bad_tensor():
    spec, cfg, pl, grads_o, new_o = _setup()
    rt = _fake_runtime(spec, cfg, pl, grads_o, new_o)
    report = []
    assert compare_shards(spec, cfg, pl, rt, grads_o, new_o, report=report) == []
    names = {(r[1], r[2]) for r in report}
    assert ("b_proj", 0) in names and ("ln2_b", 1) in names and ("wpe", None) in names
    # bf16-level noise everywhere still passes
    g = torch.Generator().manual_seed(1)
    for s, c in rt.captured.items():
        rt.captured[s] = c * (1 + 4e-3 * torch.randn(c.shape, generator=g))
    assert compare_shards(spec, cfg, pl, rt, grads_o, new_o) == []
    for bad, how in ((("b_proj", 0), "zero"), (("ln2_b", 1), "neg"), (("ln1_g", 3), "scale")):
        rt = _fake_runtime(spec, cfg, pl, grads_o, new_o)
        s = next(s for s in rt.stages if any((sl.name, sl.layer) == bad for sl in rt.stages[s].lay.slots))
        sl = rt.stages[s].lay.slot(*bad)
        piece = rt.captured[s][sl.offset:sl.offset + sl.numel]
        if how == "zero":
            piece.zero_()
        elif how == "neg":
            piece.neg_()
        else:
            piece.mul_(1.2)
        fails = compare_shards(spec, cfg, pl, rt, grads_o, new_o)
        assert any(f"{bad[0]}[{bad[1]}]" in f for f in fails), (bad, fails)
