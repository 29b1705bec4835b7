"""Shared harness: run engine steps for one rank and compare against the CPU oracle.

Used by test_engine_gpu.py (single GPU, in-process) and dist_worker.py (one
process per GPU under torchrun).  Tolerances (stated once, used everywhere):

* loss per step:       |engine - oracle| / oracle <= 1e-2  (bf16 engine vs fp32 oracle)
* grad shards:         cosine >= 0.999 and max|diff| <= 3e-2 * max|g_oracle| per stage, AND per
                       tensor piece (every named slot of the shard: weights, biases, LN gamma/beta,
                       wte/wpe, head): cosine >= 0.99 and max|diff| <= 5e-2 * max|g_oracle piece|
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
GRAD_MAXABS = 3e-2  # was 2e-2: LLaMA-7B width at s=4096 measured 2.15% (RMSNorm gain / embedding sums over 8192 tokens)
TENSOR_COS = 0.99
TENSOR_MAXABS = 5e-2


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


def params_from_flat(spec, cfg, pl, flats: dict) -> dict:
    """Named fp32 tensors from whole flat stage buffers {stage: [numel]} (P x D = 1 x 1 runs:
    the rank's fp32 master IS the whole stage).  Used by the production-width tests, whose
    initial parameters are the engine's own masters before step 1; ``zpp_init_param`` is pinned
    bit-exact to ``oracle.init_oracle`` separately (test_init_param_bit_exact) and spot-checked
    per tensor by ``check_init_sample``."""
    params = {}
    for s, flat in flats.items():
        lay = stage_layout(spec, s, cfg.num_stages, pl.stage_to_layers[s], cfg.dp_size, optimizer_sub(cfg))
        assert flat.numel() == lay.numel
        for slot in lay.slots:
            params[(slot.name, slot.layer)] = flat[slot.offset:slot.offset + slot.numel].view(*slot.shape).clone()
    return params


def check_init_sample(spec, cfg, pl, params: dict, n: int = 4096) -> list[str]:
    """The first and last ``n`` elements of every tensor equal the numpy initialiser bit for bit."""
    fails = []
    for s in range(cfg.num_stages):
        lay = stage_layout(spec, s, cfg.num_stages, pl.stage_to_layers[s], cfg.dp_size, optimizer_sub(cfg))
        for slot in lay.slots:
            t = params[(slot.name, slot.layer)].reshape(-1).cpu()
            for lo in (0, max(0, slot.numel - n)):
                cnt = min(n, slot.numel - lo)
                ref = torch.from_numpy(init_values(cnt, spec.seed, init_offset(slot.uid) + lo, slot.mean, slot.std))
                if not torch.equal(t[lo:lo + cnt], ref):
                    fails.append(f"init {slot.name}[{slot.layer}] @ {lo}")
    return fails


def flat_stage(spec, cfg, pl, s: int, named: dict) -> torch.Tensor:
    lay = stage_layout(spec, s, cfg.num_stages, pl.stage_to_layers[s], cfg.dp_size, optimizer_sub(cfg))
    dev = next(iter(named.values())).device
    out = torch.zeros(lay.numel, device=dev)
    for slot in lay.slots:
        out[slot.offset:slot.offset + slot.numel] = named[(slot.name, slot.layer)].reshape(-1)
    return out


def rank_tokens(tokens_step: torch.Tensor, z: int):
    """tokens_step [n*D, B, b, s+1] -> (ids, labels) int64 [B, b*s] of data-parallel
    rank z (= node * D + ZeRO index)."""
    t = tokens_step[z]
    B = t.shape[0]
    return t[:, :, :-1].reshape(B, -1).contiguous(), t[:, :, 1:].reshape(B, -1).contiguous()


def run_engine_step(spec, P, D, B, U, V, rank=0, world=1, steps=1, timeline=True, snapshot_init=False,
                    rt_kw=None, **cfg_kw):
    model, cfg, pl, sched = build(spec, P, D, B, U, V, **cfg_kw)
    rt = Runtime(spec, model, cfg, pl, sched, rank=rank, world=world, timeline=timeline, **(rt_kw or {}))
    if snapshot_init:  # fp32 masters before step 1 (whole stages when P x D = 1 x 1)
        torch.cuda.synchronize()
        rt.init_master = {s: st.master.clone() for s, st in rt.stages.items()}
    tokens = make_tokens(steps, cfg.inter_node_dp * D, B, spec.microbatch_samples, spec.seq_len, spec.vocab)
    out = []
    for k in range(steps):
        ids, labels = (x.cuda() for x in rank_tokens(tokens[k], rt.dp_index))
        rt.capture_grads = k == 0
        res = execute(sched, model, cfg, pl, rt, ids, labels)
        out.append(res)
    torch.cuda.synchronize()  # an overlapped step tail (AdamW on the opt stream) may still run
    return rt, (model, cfg, pl, sched), tokens, out


def oracle_for(spec, cfg, pl, tokens_step, params=None, device="cpu"):
    """Oracle step over the global batch.  ``device="cuda"`` evaluates the same fp32 code on
    the GPU with TF32 disabled (strict fp32 matmuls) - used at production widths, where the CPU
    step takes minutes; test_oracle_device_independent checks both devices agree."""
    D, B, b, s1 = tokens_step.shape
    ids = tokens_step[:, :, :, :-1].reshape(D * B * b, s1 - 1).to(device)
    labels = tokens_step[:, :, :, 1:].reshape(D * B * b, s1 - 1).to(device)
    if params is None:
        params = oracle_params(spec, cfg, pl)
    params = {k: v.to(device) for k, v in params.items()}
    if device != "cpu":
        torch.backends.cuda.matmul.allow_tf32 = False
        torch.backends.cudnn.allow_tf32 = False
    return oracle_step(params, ids, labels, layers=spec.num_layers, heads=spec.heads, lr=spec.lr,
                       betas=(spec.beta1, spec.beta2), eps=spec.adam_eps,
                       weight_decay=spec.weight_decay, ln_eps=spec.ln_eps, arch=spec.arch,
                       rope_base=spec.rope_base)


def tensor_grad_report(st, lo: int, g: torch.Tensor, g_ref: torch.Tensor) -> list[tuple]:
    """(name, layer, cos, maxdiff, max|g_ref|, ok) for every tensor piece of shard range
    [lo, lo + len(g)) of the stage layout; exact-zero oracle pieces are skipped."""
    out = []
    hi = lo + g.numel()
    for slot in st.lay.slots:
        a, b = max(lo, slot.offset), min(hi, slot.offset + slot.numel)
        if a >= b:
            continue
        x, r = g[a - lo:b - lo], g_ref[a - lo:b - lo]
        rmax = r.abs().max().item()
        if rmax == 0.0:
            continue
        cos = torch.nn.functional.cosine_similarity(x, r, dim=0).item() if b - a > 1 else 1.0
        maxd = (x - r).abs().max().item()
        ok = (cos >= TENSOR_COS or b - a == 1) and maxd <= TENSOR_MAXABS * rmax
        out.append((slot.name, slot.layer, cos, maxd, rmax, ok))
    return out


def compare_shards(spec, cfg, pl, rt, grads_o, new_o, report=None) -> list[str]:
    """Return a list of failures (empty = pass) for this rank's stages.  ``report`` (a list)
    receives every per-tensor (stage, name, layer, cos, maxdiff, max|g|, ok) row."""
    fails = []
    lr, wd = spec.lr, spec.weight_decay
    for s, st in rt.stages.items():
        ns, nsub = st.lay.shard_numel, st.nsub   # ZeRO-1 outer mode: Adam state of sub-shard `node`
        lo = rt.z * ns + (rt.node * nsub if st.sub > 1 else 0)
        sl = slice(lo, lo + nsub)
        g_ref = flat_stage(spec, cfg, pl, s, grads_o)[sl]
        dev = g_ref.device
        g = rt.captured[s].float().to(dev)
        cos = torch.nn.functional.cosine_similarity(g, g_ref, dim=0).item()
        maxd = (g - g_ref).abs().max().item()
        if cos < GRAD_COS or maxd > GRAD_MAXABS * g_ref.abs().max().item():
            fails.append(f"stage {s} grad: cos={cos:.6f} maxdiff={maxd:.3e} max|g|={g_ref.abs().max():.3e}")
        for name, layer, tcos, tmax, rmax, ok in tensor_grad_report(st, lo, g, g_ref):
            if report is not None:
                report.append((s, name, layer, tcos, tmax, rmax, ok))
            if not ok:
                fails.append(f"stage {s} grad {name}[{layer}]: cos={tcos:.6f} maxdiff={tmax:.3e} max|g|={rmax:.3e}")
        p_ref = flat_stage(spec, cfg, pl, s, new_o)[sl]
        p = st.master.float().to(dev)
        d = (p - p_ref).abs()
        bound = 2 * lr + lr * wd * p_ref.abs() + 1e-7
        tight = (d <= 0.1 * lr).float().mean().item()
        if (d > bound).any() or tight < 0.99:
            fails.append(f"stage {s} master: max|d|={d.max():.3e} frac<=0.1lr={tight:.4f}")
        if not torch.equal(st.sub_bf16, st.master.to(torch.bfloat16)):
            fails.append(f"stage {s}: bf16 shard != rne(master)")
        if st.sub > 1:  # AG_PARAM_INTER: the whole bf16 shard is every replica's update
            full = flat_stage(spec, cfg, pl, s, new_o)[rt.z * ns:(rt.z + 1) * ns]
            d = (st.shard_bf16.float().to(dev) - full).abs()
            if (d > 2 * lr + lr * wd * full.abs() + 1e-2 * full.abs() + 1e-6).any():
                fails.append(f"stage {s}: gathered bf16 shard off by {d.max():.3e}")
    return fails
