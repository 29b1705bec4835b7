"""CPU fp32 oracle of one ZeroPP training step.

TEST INFRASTRUCTURE ONLY - imported by tests/, __graft_entry__.smoke() and the
bench ``cpu_baseline`` / ``--impl reference`` legs as the checker or the CPU
baseline; never imported by the product path.

Parity status: the reference package (`pkg/src/zeroppsim`) contains NO step
arithmetic - it is a schedule simulator (`SPEC.md:15,89`).
Loss / gradient / parameter parity is therefore *unpinned by the reference*; this
oracle is the engine-independent restatement of the step semantics the
reference's schedule implies:

* every (stage, micro-batch) runs F then B then W (`schedules.py:98-141`); the
  loss is folded into F of the last stage (`SPEC.md:170`);
* gradients accumulate over the U micro-batches of a unit and are summed over
  the D ranks of the ZeRO group by RS_GRAD (`schedules.py:76-78`,
  `PAPER.md:177,253`); since summation order only changes rounding, the oracle
  computes one fp32 forward/backward over the GLOBAL batch (D x B micro-batches);
* OPT runs after every reduction (`schedules.py:144-163`): AdamW with
  torch.optim.AdamW semantics on fp32 master weights.

The model is the GPT-2 style pre-LN decoder the engine runs (untied LM head,
tanh GeLU, causal attention, loss = mean token cross-entropy), or the LLaMA
block of BASELINE config C4 (RMSNorm, SwiGLU, rotate-half RoPE, no biases, no
learned positions; ``llama_forward_loss``).
"""

from __future__ import annotations

import math

import torch
import torch.nn.functional as F


def gpt_forward_loss(params: dict, ids: torch.Tensor, labels: torch.Tensor, *, layers: int, heads: int,
                     eps: float = 1e-5) -> torch.Tensor:
    """Mean cross-entropy over all tokens. ``ids``/``labels``: int64 [N, s]."""
    N, s = ids.shape
    wte, wpe = params[("wte", None)], params[("wpe", None)]
    h = wte.shape[1]
    dh = h // heads
    x = wte[ids] + wpe[torch.arange(s, device=ids.device)][None]
    mask = torch.ones(s, s, dtype=torch.bool, device=ids.device).triu(1)
    for l in range(layers):
        p = lambda n: params[(n, l)]  # noqa: E731
        xn = F.layer_norm(x, (h,), p("ln1_g"), p("ln1_b"), eps)
        qkv = xn @ p("w_qkv").t() + p("b_qkv")
        q, k, v = qkv.view(N, s, 3, heads, dh).unbind(2)
        q, k, v = (t.transpose(1, 2) for t in (q, k, v))
        att = (q @ k.transpose(-1, -2)) / math.sqrt(dh)
        att = att.masked_fill(mask, float("-inf")).softmax(-1)
        o = (att @ v).transpose(1, 2).reshape(N, s, h)
        x = x + o @ p("w_proj").t() + p("b_proj")
        xn = F.layer_norm(x, (h,), p("ln2_g"), p("ln2_b"), eps)
        u = xn @ p("w_fc1").t() + p("b_fc1")
        x = x + F.gelu(u, approximate="tanh") @ p("w_fc2").t() + p("b_fc2")
    xf = F.layer_norm(x, (h,), params[("lnf_g", None)], params[("lnf_b", None)], eps)
    logits = xf @ params[("w_lm", None)].t()
    return F.cross_entropy(logits.view(N * s, -1), labels.reshape(-1))


def _rms(x, g, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * g


def _rope(t, base: float):
    """Rotate-half RoPE of t [N, H, s, d] at positions 0..s-1."""
    s, d = t.shape[-2], t.shape[-1]
    inv = torch.exp2(-(2.0 * torch.arange(d // 2, dtype=torch.float32, device=t.device) / d) * math.log2(base))
    ang = torch.arange(s, dtype=torch.float32, device=t.device)[:, None] * inv[None]
    cos, sin = ang.cos(), ang.sin()
    a, b = t[..., : d // 2], t[..., d // 2:]
    return torch.cat([a * cos - b * sin, b * cos + a * sin], dim=-1)


def llama_forward_loss(params: dict, ids: torch.Tensor, labels: torch.Tensor, *, layers: int, heads: int,
                       eps: float = 1e-5, rope_base: float = 10000.0) -> torch.Tensor:
    """LLaMA block: x += Wo attn(rope(q), rope(k), v)(rms(x));
    x += Wdown (silu(gate) * up)(rms(x)) with [gate; up] = w_fc1 rms(x)."""
    N, s = ids.shape
    wte = params[("wte", None)]
    h = wte.shape[1]
    dh = h // heads
    x = wte[ids]
    mask = torch.ones(s, s, dtype=torch.bool, device=ids.device).triu(1)
    for l in range(layers):
        p = lambda n: params[(n, l)]  # noqa: E731
        qkv = _rms(x, p("ln1_g"), eps) @ p("w_qkv").t()
        q, k, v = qkv.view(N, s, 3, heads, dh).unbind(2)
        q, k, v = (t.transpose(1, 2) for t in (q, k, v))
        q, k = _rope(q, rope_base), _rope(k, rope_base)
        att = (q @ k.transpose(-1, -2)) / math.sqrt(dh)
        att = att.masked_fill(mask, float("-inf")).softmax(-1)
        o = (att @ v).transpose(1, 2).reshape(N, s, h)
        x = x + o @ p("w_proj").t()
        gate, up = (_rms(x, p("ln2_g"), eps) @ p("w_fc1").t()).chunk(2, dim=-1)
        x = x + (F.silu(gate) * up) @ p("w_fc2").t()
    xf = _rms(x, params[("lnf_g", None)], eps)
    logits = xf @ params[("w_lm", None)].t()
    return F.cross_entropy(logits.view(N * s, -1), labels.reshape(-1))


def oracle_step(params: dict, ids: torch.Tensor, labels: torch.Tensor, *, layers: int, heads: int,
                lr: float, betas=(0.9, 0.95), eps: float = 1e-8, weight_decay: float = 0.1,
                ln_eps: float = 1e-5, threads: int | None = None, arch: str = "gpt",
                rope_base: float = 10000.0):
    """One step: returns (loss, grads dict, updated params dict), all fp32 CPU."""
    if threads:
        torch.set_num_threads(threads)
    leaf = {k: v.detach().clone().float().requires_grad_(True) for k, v in params.items()}
    if arch == "llama":
        loss = llama_forward_loss(leaf, ids, labels, layers=layers, heads=heads, eps=ln_eps, rope_base=rope_base)
    else:
        loss = gpt_forward_loss(leaf, ids, labels, layers=layers, heads=heads, eps=ln_eps)
    loss.backward()
    grads = {k: v.grad.detach().clone() for k, v in leaf.items()}
    opt = torch.optim.AdamW(list(leaf.values()), lr=lr, betas=betas, eps=eps, weight_decay=weight_decay,
                            foreach=False)
    opt.step()
    new = {k: v.detach().clone() for k, v in leaf.items()}
    return loss.item(), grads, new


def make_tokens(steps: int, D: int, B: int, b: int, s: int, vocab: int, seed: int = 20240817) -> torch.Tensor:
    """Synthetic tokens int64 [steps, D, B, b, s+1] from one CPU generator
    (seed = the reference's DEFAULT_FUZZ_SEED, `cli.py:26`)."""
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, vocab, (steps, D, B, b, s + 1), generator=g)
