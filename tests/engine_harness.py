"""Shared harness: run engine steps for one rank and compare against the CPU oracle.

Used by test_engine_gpu.py (single GPU, in-process) and dist_worker.py (one
process per GPU under torchrun).  Tolerances (stated once, used everywhere):

* loss per step:       |engine - oracle| / oracle <= 1e-2  (bf16 engine vs fp32 oracle)
* grad shards:         cosine >= 0.999 and max|diff| <= 2e-2 * max|g_oracle| per stage
* master after AdamW:  |diff| <= 2*lr + lr*wd*|theta| everywhere and <= 0.1*lr on >= 99%
* bf16 param shard == round-to-nearest-even(master) exactly
"""

from __future__ import annotations

import torch

from oracle.gpt_oracle import make_tokens, oracle_step
from oracle.init_oracle import init_values
from paper_2402_03791_b200 import ModelSpec, ParallelConfig, generate, make_placement
from paper_2402_03791_b200.engine import GPTSpec, Runtime, execute
from paper_2402_03791_b200.engine.model import init_offset, optimizer_sub, stage_layout

LOSS_RTOL = 1e-2
GRAD_COS = 0.999
GRAD_MAXABS = 2e-2


def build(spec: GPTSpec, P: int, D: int, B: int, U: int, V: int, **cfg_kw):
    model = ModelSpec(num_layers=spec.num_layers, hidden_size=spec.hidden, seq_len=spec.seq_len)
    cfg = ParallelConfig(pp_size=P, dp_size=D, microbatches=B, unit_size=U, stages_per_device=V,
                         microbatch_samples=spec.microbatch_samples, **cfg_kw)
    pl = make_placement(cfg, model)
    return model, cfg, pl, generate(model, cfg, pl)


def oracle_params(spec: GPTSpec, cfg, pl) -> dict:
    params = {}
    for s in range(cfg.num_stages):
        lay = stage_layout(spec, s, cfg.num_stages, pl.stage_to_layers[s], cfg.dp_size, optimizer_sub(cfg))
        for slot in lay.slots:
            v = init_values(slot.numel, spec.seed, init_offset(slot.uid), slot.mean, slot.std)
            params[(slot.name, slot.layer)] = torch.from_numpy(v).view(*slot.shape)
    return params


def flat_stage(spec, cfg, pl, s: int, named: dict) -> torch.Tensor:
    lay = stage_layout(spec, s, cfg.num_stages, pl.stage_to_layers[s], cfg.dp_size, optimizer_sub(cfg))
    out = torch.zeros(lay.numel)
    for slot in lay.slots:
        out[slot.offset:slot.offset + slot.numel] = named[(slot.name, slot.layer)].reshape(-1)
    return out


def rank_tokens(tokens_step: torch.Tensor, z: int):
    """tokens_step [n*D, B, b, s+1] -> (ids, labels) int64 [B, b*s] of data-parallel
    rank z (= node * D + ZeRO index)."""
    t = tokens_step[z]
    B = t.shape[0]
    return t[:, :, :-1].reshape(B, -1).contiguous(), t[:, :, 1:].reshape(B, -1).contiguous()


def run_engine_step(spec, P, D, B, U, V, rank=0, world=1, steps=1, timeline=True, **cfg_kw):
    model, cfg, pl, sched = build(spec, P, D, B, U, V, **cfg_kw)
    rt = Runtime(spec, model, cfg, pl, sched, rank=rank, world=world, timeline=timeline)
    tokens = make_tokens(steps, cfg.inter_node_dp * D, B, spec.microbatch_samples, spec.seq_len, spec.vocab)
    out = []
    for k in range(steps):
        ids, labels = (x.cuda() for x in rank_tokens(tokens[k], rt.dp_index))
        rt.capture_grads = k == 0
        res = execute(sched, model, cfg, pl, rt, ids, labels)
        out.append(res)
    return rt, (model, cfg, pl, sched), tokens, out


def oracle_for(spec, cfg, pl, tokens_step):
    D, B, b, s1 = tokens_step.shape
    ids = tokens_step[:, :, :, :-1].reshape(D * B * b, s1 - 1)
    labels = tokens_step[:, :, :, 1:].reshape(D * B * b, s1 - 1)
    params = oracle_params(spec, cfg, pl)
    return oracle_step(params, ids, labels, layers=spec.num_layers, heads=spec.heads, lr=spec.lr,
                       betas=(spec.beta1, spec.beta2), eps=spec.adam_eps,
                       weight_decay=spec.weight_decay, ln_eps=spec.ln_eps, arch=spec.arch,
                       rope_base=spec.rope_base)


def compare_shards(spec, cfg, pl, rt, grads_o, new_o) -> list[str]:
    """Return a list of failures (empty = pass) for this rank's stages."""
    fails = []
    lr, wd = spec.lr, spec.weight_decay
    for s, st in rt.stages.items():
        ns, nsub = st.lay.shard_numel, st.nsub   # ZeRO-1 outer mode: Adam state of sub-shard `node`
        lo = rt.z * ns + (rt.node * nsub if st.sub > 1 else 0)
        sl = slice(lo, lo + nsub)
        g_ref = flat_stage(spec, cfg, pl, s, grads_o)[sl]
        g = rt.captured[s].float().cpu()
        cos = torch.nn.functional.cosine_similarity(g, g_ref, dim=0).item()
        maxd = (g - g_ref).abs().max().item()
        if cos < GRAD_COS or maxd > GRAD_MAXABS * g_ref.abs().max().item():
            fails.append(f"stage {s} grad: cos={cos:.6f} maxdiff={maxd:.3e} max|g|={g_ref.abs().max():.3e}")
        p_ref = flat_stage(spec, cfg, pl, s, new_o)[sl]
        p = st.master.float().cpu()
        d = (p - p_ref).abs()
        bound = 2 * lr + lr * wd * p_ref.abs() + 1e-7
        tight = (d <= 0.1 * lr).float().mean().item()
        if (d > bound).any() or tight < 0.99:
            fails.append(f"stage {s} master: max|d|={d.max():.3e} frac<=0.1lr={tight:.4f}")
        if not torch.equal(st.sub_bf16.cpu(), st.master.to(torch.bfloat16).cpu()):
            fails.append(f"stage {s}: bf16 shard != rne(master)")
        if st.sub > 1:  # AG_PARAM_INTER: the whole bf16 shard is every replica's update
            full = flat_stage(spec, cfg, pl, s, new_o)[rt.z * ns:(rt.z + 1) * ns]
            d = (st.shard_bf16.float().cpu() - full).abs()
            if (d > 2 * lr + lr * wd * full.abs() + 1e-2 * full.abs() + 1e-6).any():
                fails.append(f"stage {s}: gathered bf16 shard off by {d.max():.3e}")
    return fails
