"""Model description (GPT or LLaMA block) and the flat, ZeRO-shardable parameter
layout of a stage.

The reference models a stage only as ``layers * M_w`` bytes (ModelSpec,
`config.py:36-89`; stage bytes `schedules.py:45-49`).  The engine needs the
real tensors: a GPT-2 style pre-LN decoder (untied LM head, tanh GeLU,
causal attention) whose parameters for each pipeline stage live in ONE flat
bf16 buffer, so that a stage's ZeRO-3 all-gather / reduce-scatter is a single
NCCL call on a contiguous range (AG_PARAM / RS_GRAD, `schedules.py:72-78`).

Layout of stage s with layers [lo, hi) (each tensor 64-element aligned):
    s == 0   : wte [V, h], wpe [S, h]
    per layer: ln1_g, ln1_b, w_qkv [3h, h], b_qkv, w_proj [h, h], b_proj,
               ln2_g, ln2_b, w_fc1 [4h, h], b_fc1, w_fc2 [h, 4h], b_fc2
    s == S-1 : lnf_g, lnf_b, w_lm [V, h]
LLaMA (``arch="llama"``: RMSNorm, SwiGLU, RoPE, no biases):
    s == 0   : wte [V, h]
    per layer: ln1_g, w_qkv [3h, h], w_proj [h, h], ln2_g, w_fc1 [2f, h] (= [gate; up]),
               w_fc2 [h, f]
    s == S-1 : lnf_g, w_lm [V, h]
The flat size is padded to a multiple of 64*D (64*D*n in ZeRO-1 outer mode) so every
ZeRO shard (and optimizer sub-shard) is 128-byte aligned.  Shard z of D owns elements
[z*n/D, (z+1)*n/D).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

ALIGN = 64

LAYER_TENSORS = ("ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_proj", "b_proj",
                 "ln2_g", "ln2_b", "w_fc1", "b_fc1", "w_fc2", "b_fc2")
LLAMA_LAYER_TENSORS = ("ln1_g", "w_qkv", "w_proj", "ln2_g", "w_fc1", "w_fc2")
ARCHS = ("gpt", "llama")


@dataclass(frozen=True)
class GPTSpec:
    """Engine-side model + optimizer settings (the reference config has no such
    section, SURVEY.md section 5 'config / flag system')."""

    num_layers: int
    hidden: int
    heads: int
    seq_len: int
    vocab: int = 50304
    microbatch_samples: int = 1
    ln_eps: float = 1e-5
    init_std: float = 0.02
    seed: int = 20240817
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.95
    adam_eps: float = 1e-8
    weight_decay: float = 0.1
    arch: str = "gpt"                # "gpt" (pre-LN, GeLU, learned positions) | "llama"
    ffn_hidden: int | None = None    # MLP width; default 4h (GPT)
    rope_base: float = 10000.0       # LLaMA rotary base

    def __post_init__(self):
        if self.arch not in ARCHS:
            raise ValueError(f"arch must be one of {ARCHS}")
        if self.ffn % 64:
            raise ValueError("ffn_hidden must be a multiple of 64")
        if self.hidden % self.heads:
            raise ValueError("hidden must be divisible by heads")
        if self.head_dim not in (64, 128):
            raise ValueError("head_dim must be 64 or 128 (attention kernels)")
        if self.seq_len % 128:
            raise ValueError("seq_len must be a multiple of 128 (attention tiles)")
        if self.hidden % 64 or self.vocab % 64:
            raise ValueError("hidden and vocab must be multiples of 64")

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    @property
    def ffn(self) -> int:
        return self.ffn_hidden or 4 * self.hidden

    @property
    def llama(self) -> bool:
        return self.arch == "llama"

    @property
    def tokens_per_microbatch(self) -> int:
        return self.microbatch_samples * self.seq_len

    def flops_per_token(self) -> float:
        """Model FLOPs per token (fwd+bwd, attention at full s^2)."""
        L, h, s, V = self.num_layers, self.hidden, self.seq_len, self.vocab
        if self.llama:
            return 6.0 * L * (4.0 * h * h + 3.0 * h * self.ffn) + 12.0 * L * s * h + 6.0 * h * V
        return 72.0 * L * h * h + 12.0 * L * s * h + 6.0 * h * V

    def num_params(self) -> int:
        h, L, V, S = self.hidden, self.num_layers, self.vocab, self.seq_len
        if self.llama:
            return L * (4 * h * h + 3 * h * self.ffn + 2 * h) + V * h + h + V * h
        per_layer = 12 * h * h + 13 * h
        return L * per_layer + V * h + S * h + 2 * h + V * h

    @classmethod
    def gpt_6p2b(cls, **kw) -> "GPTSpec":
        return cls(num_layers=32, hidden=4096, heads=32, seq_len=2048, **kw)

    @classmethod
    def gpt_1p3b(cls, **kw) -> "GPTSpec":
        return cls(num_layers=24, hidden=2048, heads=16, seq_len=2048, **kw)

    @classmethod
    def gpt_13b(cls, **kw) -> "GPTSpec":
        """SURVEY.md C5 / BASELINE configs[4]: L40 h5120 a40 (head_dim 128) s2048, 13.1 B params:
        236 GB of fp32 master + Adam + bf16 state (18 B/param), so it needs P x D >= 2 on 180 GB B200s."""
        return cls(num_layers=40, hidden=5120, heads=40, seq_len=2048, **kw)

    @classmethod
    def tiny(cls, **kw) -> "GPTSpec":
        return cls(num_layers=4, hidden=256, heads=4, seq_len=128, **kw)

    @classmethod
    def llama_7b(cls, **kw) -> "GPTSpec":
        """L32 h4096 a32 s4096, SwiGLU ffn 11008, vocab 32000, RoPE, untied."""
        return cls(num_layers=32, hidden=4096, heads=32, seq_len=4096, vocab=32000, arch="llama",
                   ffn_hidden=11008, **kw)

    @classmethod
    def tiny_llama(cls, **kw) -> "GPTSpec":
        return cls(num_layers=4, hidden=256, heads=4, seq_len=128, vocab=32000, arch="llama",
                   ffn_hidden=704, **kw)


@dataclass(frozen=True)
class TensorSlot:
    name: str
    layer: int | None          # global layer index (None for embedding / head)
    shape: tuple[int, ...]
    offset: int                # element offset in the flat stage buffer
    uid: int                   # global tensor id, seeds the initialiser
    mean: float
    std: float

    @property
    def numel(self) -> int:
        return math.prod(self.shape)


def _align(n: int, a: int = ALIGN) -> int:
    return (n + a - 1) // a * a


@dataclass
class StageLayout:
    stage: int
    layers: tuple[int, int]
    slots: list[TensorSlot] = field(default_factory=list)
    numel: int = 0          # padded flat size
    shard_numel: int = 0

    def slot(self, name: str, layer: int | None = None) -> TensorSlot:
        for s in self.slots:
            if s.name == name and s.layer == layer:
                return s
        raise KeyError((name, layer))


def stage_layout(spec: GPTSpec, stage: int, num_stages: int, layer_range: tuple[int, int],
                 dp: int, sub: int = 1) -> StageLayout:
    """``sub`` > 1 (ZeRO-1 outer mode, n nodes) additionally makes every shard split
    into ``sub`` equal, 128-byte aligned optimizer sub-shards."""
    h, V, L = spec.hidden, spec.vocab, spec.num_layers
    std, proj_std = spec.init_std, spec.init_std / math.sqrt(2.0 * L)
    lay = StageLayout(stage, layer_range)
    off = 0

    def add(name, layer, shape, uid, mean=0.0, sd=0.0):
        nonlocal off
        slot = TensorSlot(name, layer, tuple(shape), off, uid, mean, sd)
        lay.slots.append(slot)
        off = _align(off + slot.numel)

    if spec.llama:
        f = spec.ffn
        if stage == 0:
            add("wte", None, (V, h), 1, sd=std)
        for l in range(*layer_range):
            base = 16 + 16 * l
            shapes = {"ln1_g": (h,), "w_qkv": (3 * h, h), "w_proj": (h, h), "ln2_g": (h,),
                      "w_fc1": (2 * f, h), "w_fc2": (h, f)}
            for name in LLAMA_LAYER_TENSORS:
                uid = base + LAYER_TENSORS.index(name)
                if name.endswith("_g"):
                    add(name, l, shapes[name], uid, mean=1.0)
                else:
                    add(name, l, shapes[name], uid, sd=proj_std if name in ("w_proj", "w_fc2") else std)
        if stage == num_stages - 1:
            add("lnf_g", None, (h,), 3, mean=1.0)
            add("w_lm", None, (V, h), 5, sd=std)
        lay.numel = _align(off, ALIGN * dp * sub)
        lay.shard_numel = lay.numel // dp
        return lay
    if stage == 0:
        add("wte", None, (V, h), 1, sd=std)
        add("wpe", None, (spec.seq_len, h), 2, sd=std)
    for l in range(*layer_range):
        base = 16 + 16 * l
        shapes = {"ln1_g": (h,), "ln1_b": (h,), "w_qkv": (3 * h, h), "b_qkv": (3 * h,),
                  "w_proj": (h, h), "b_proj": (h,), "ln2_g": (h,), "ln2_b": (h,),
                  "w_fc1": (4 * h, h), "b_fc1": (4 * h,), "w_fc2": (h, 4 * h), "b_fc2": (h,)}
        for j, name in enumerate(LAYER_TENSORS):
            if name.endswith("_g"):
                add(name, l, shapes[name], base + j, mean=1.0)
            elif name.startswith("w_"):
                add(name, l, shapes[name], base + j, sd=proj_std if name in ("w_proj", "w_fc2") else std)
            else:
                add(name, l, shapes[name], base + j)
    if stage == num_stages - 1:
        add("lnf_g", None, (h,), 3, mean=1.0)
        add("lnf_b", None, (h,), 4)
        add("w_lm", None, (V, h), 5, sd=std)
    lay.numel = _align(off, ALIGN * dp * sub)
    lay.shard_numel = lay.numel // dp
    return lay


def optimizer_sub(cfg) -> int:
    """Optimizer sub-shards per ZeRO shard: n in ZeRO-1 outer mode (RS_GRAD_INTER /
    AG_PARAM_INTER, `schedules.py:425-427`), else 1 (DP outer mode replicates Adam)."""
    from ..config import HybridMode
    return cfg.inter_node_dp if cfg.hybrid_mode is HybridMode.ZERO1_OUTER else 1


def init_offset(uid: int) -> int:
    """Counter base of a tensor for the deterministic initialiser (2^40 per tensor)."""
    return uid << 40


def shard_init_ranges(lay: StageLayout, z: int):
    """(slot, start_in_tensor, start_in_shard, count) for every tensor piece in shard z."""
    lo, hi = z * lay.shard_numel, (z + 1) * lay.shard_numel
    for slot in lay.slots:
        a, b = max(lo, slot.offset), min(hi, slot.offset + slot.numel)
        if a < b:
            yield slot, a - slot.offset, a - lo, b - a


def nccl_bytes_per_step(spec: GPTSpec, cfg, placement, sched, p: int, rs_wire: str = "bf16") -> tuple[int, int]:
    """(intra, inter) bytes pipeline rank ``p`` receives through NCCL in one step, task by task
    as the executor issues them (ring collectives: an all-gather / reduce-scatter over g ranks
    moves (g-1)/g of the full buffer per rank, an all-reduce twice that):

    * AG_PARAM, RS_GRAD (`schedules.py:72-78`): (D-1) x shard x 2 B of the stage's flat bf16
      buffer -- the reference's ``((D-1)/D) * M_w * layers`` with the stage's real size
      (RS_GRAD x 4 B with ``rs_wire="fp32"``);
    * AR_GRAD (`:80-81`): 2 (n-1)/n x shard x 2 B per local stage;
    * RS_GRAD_INTER / AG_PARAM_INTER (`:83-87`): (n-1) x optimizer sub-shard x 2 B per stage.
    ``StepResult.nccl_bytes_intra/inter`` must equal this (tests/test_engine_gpu.py via
    dist_worker.py); tests/test_comm_bytes.py relates it to the reference's own byte model."""
    from ..tasks import TaskKind
    D, n, S = cfg.dp_size, cfg.inter_node_dp, cfg.num_stages
    sub = optimizer_sub(cfg)
    lays = {s: stage_layout(spec, s, S, placement.stage_to_layers[s], D, sub) for s in placement.device_stages(p)}
    intra = inter = 0
    for t in sched.per_device[p]:
        if t.kind is TaskKind.AG_PARAM:
            intra += (D - 1) * lays[t.stage].shard_numel * 2
        elif t.kind is TaskKind.RS_GRAD:
            intra += (D - 1) * lays[t.stage].shard_numel * (4 if rs_wire == "fp32" else 2)
        elif t.kind is TaskKind.AR_GRAD and n > 1:
            inter += sum(2 * (n - 1) * lay.shard_numel * 2 // n for lay in lays.values())
        elif t.kind in (TaskKind.RS_GRAD_INTER, TaskKind.AG_PARAM_INTER) and n > 1:
            inter += sum((n - 1) * (lay.shard_numel // sub) * 2 for lay in lays.values())
    return intra, inter


def memory_estimate(spec: GPTSpec, model, cfg, placement, sched, p: int) -> tuple[float, float]:
    """(static, activation) bytes pipeline rank ``p`` will hold at peak.

    static: per local stage the gathered bf16 stage (2 B/param), the fp32 master / exp_avg /
    exp_avg_sq / shard grad (16 B per shard param) and, at D > 1, the fp32 full-stage grad.
    activations: the reference simulator's live-micro-batch peak (`simulation.py:219-280`)
    with the engine's real per-layer stash (planner.engine_memory_model).  Measured peaks are
    1-9 GB above this (GEMM workspaces, logits, NCCL buffers; profiles/r02)."""
    import dataclasses
    from ..config import CommCostModel
    from ..planner import engine_memory_model
    from ..simulation import simulate
    D = cfg.dp_size
    static = 0
    for s in placement.device_stages(p):
        n = stage_layout(spec, s, cfg.num_stages, placement.stage_to_layers[s], D, optimizer_sub(cfg)).numel
        static += 2 * n + 16 * n // D + (4 * n if D > 1 else 0)
    fitted, _ = engine_memory_model(spec, model)
    fitted = dataclasses.replace(fitted, weight_mem_per_layer=1e-9)  # activations only
    sim = simulate(sched, fitted, dataclasses.replace(cfg, optimizer_state_multiplier=0.0), placement,
                   CommCostModel(intra_node_bandwidth=1e12, inter_node_bandwidth=1e12))
    return float(static), float(sim.peak_mem[p])
