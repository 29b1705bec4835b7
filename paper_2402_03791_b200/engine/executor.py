"""Per-rank ZeroPP step executor: the real-hardware replacement for the
reference's ``simulate`` (`pkg/src/zeroppsim/simulation.py:90-158`).

One OS process per GPU; rank r = node*P*D + p*D + z: node is the outer
data-parallel replica (``inter_node_dp`` = n "nodes"; one box emulates them), p the
pipeline rank and z the ZeRO index.  The host walks ``sched.per_device[p]`` in order and only enqueues
work; ordering across streams uses CUDA events:

    compute    F / B / W (GPT stage math, libzpp kernels), OPT (sharded AdamW)
    ag         AG_PARAM: ncclAllGather of the stage's bf16 shard (in place)
    rs         RS_GRAD : fp32 stage grad -> bf16 wire -> ncclReduceScatter -> += fp32 shard grad
               AR_GRAD / RS_GRAD_INTER: the shard grad across the n replicas (outer tail)
    ag         AG_PARAM_INTER: bf16 optimizer sub-shards -> full shard (ZeRO-1 outer mode)
    act_send / act_recv / grad_send / grad_recv: stage-boundary P2P

P2P uses one dedicated 2-rank communicator per (message kind, directed pair):
NCCL matches send/recv by order only, and a shared channel would swap
activations and gradients.  The ZeRO group uses two
communicators (one per stream) so all-gathers and reduce-scatters never share
a communicator across streams.

Task semantics follow the reference schedule exactly (task order from
`schedules.py:339-474`; edges `schedules.py:98-163`); the executor asserts the
schedule validates (`validation.py:99-135`) before touching the GPU.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import torch

from ..config import HybridMode, ModelSpec, ParallelConfig, Placement, RecomputeMode
from ..tasks import Schedule, Task, TaskKind
from ..validation import validate
from . import lib, ops
from .model import GPTSpec, StageLayout, init_offset, memory_estimate, optimizer_sub, shard_init_ranges, stage_layout

BF16, F32 = torch.bfloat16, torch.float32


def rank_coords(rank: int, n: int, P: int, D: int) -> tuple[int, int, int]:
    """rank -> (node, pipeline rank p, ZeRO index z); rank = node*P*D + p*D + z."""
    if not 0 <= rank < n * P * D:
        raise ValueError(f"rank {rank} outside n*P*D = {n * P * D}")
    node, local = divmod(rank, P * D)
    return node, local // D, local % D


def comm_plan(n: int, P: int, D: int) -> list[tuple[tuple, list[int]]]:
    """Every NCCL communicator of an n x P x D job as (key, global ranks), in the one
    global creation order all ranks follow.  Keys are node-local (each rank joins only
    its own node's): ("ag", p) / ("rs", p) = ZeRO group p (one per stream);
    ("act", p, p+1, z) / ("grad", p, p-1, z) = directed 2-rank P2P channels (ring wrap,
    `config.py:186`); ("inter",) = the n replicas of one (p, z) shard (outer tail)."""
    plan = []
    for node in range(n):
        base = node * P * D
        for p in range(P):
            grp = [base + p * D + z for z in range(D)]
            if D > 1:
                plan.append((("ag", p), grp))
                plan.append((("rs", p), grp))
        if P > 1:
            for z in range(D):
                for p in range(P):
                    nxt, prv = (p + 1) % P, (p - 1) % P
                    plan.append((("act", p, nxt, z), [base + p * D + z, base + nxt * D + z]))
                    plan.append((("grad", p, prv, z), [base + p * D + z, base + prv * D + z]))
    if n > 1:
        for local in range(P * D):
            plan.append((("inter",), [node * P * D + local for node in range(n)]))
    return plan


@dataclass
class StepResult:
    """SimResult-shaped measurement of one executed step on this rank
    (fields mirror `simulation.py:53-77`, times in milliseconds)."""

    loss_sum: torch.Tensor                  # device scalar: sum of CE over this rank's tokens
    tokens: int                             # tokens processed by this rank's last stage
    step_ms: float | None = None
    task_times: dict = field(default_factory=dict)
    exposed_comm_ms: float | None = None    # compute-stream waits on AG / RS
    p2p_wait_ms: float | None = None        # compute-stream waits on P2P recv (bubble + transfer)
    waits: list | None = None               # (kind, task_id, ms) of every timed compute-stream wait
    busy_ms: float | None = None
    sim: object = None                      # timeline runtimes: the whole-job SimResult (engine.timeline)
    # bytes this rank received through NCCL collectives this step (ring algorithms: an
    # all-gather / reduce-scatter over g ranks moves (g-1)/g of the full buffer per rank, an
    # all-reduce twice that) -- the executed counterpart of the reference's task bytes
    # (`schedules.py:72-87`), checked against them in tests/test_comm_bytes.py
    nccl_bytes_intra: int = 0
    nccl_bytes_inter: int = 0

    def __getattr__(self, name):
        # SimResult superset: makespan, per_device_busy/idle, bubble_ratios, peak_mem,
        # comm_bytes_intra/inter, ... and the extras (loss, tokens_per_s, mfu, ...)
        sim = self.__dict__.get("sim")
        if sim is not None:
            if hasattr(sim, name):
                return getattr(sim, name)
            if name in sim.extras:
                return sim.extras[name]
        raise AttributeError(name)


def opt_chunks(lay: StageLayout) -> dict:
    """Partition of the flat stage buffer [0, numel) into optimizer chunks: "embed"
    (wte, wpe), one per layer, and "head" (final norm + LM head); alignment padding goes
    with the preceding tensor.  AdamW is elementwise, so updating chunk by chunk is
    bit-identical to one launch over the whole buffer."""
    keys = []
    for sl in lay.slots:
        keys.append("embed" if sl.name in ("wte", "wpe") else
                    "head" if sl.layer is None else sl.layer)
    out: dict = {}
    for i, (sl, k) in enumerate(zip(lay.slots, keys)):
        end = lay.slots[i + 1].offset if i + 1 < len(lay.slots) else lay.numel
        lo, hi = out.get(k, (sl.offset, end))
        out[k] = (min(lo, sl.offset), max(hi, end))
    return out


class _Stage:
    """Buffers and views of one pipeline stage held by this rank.

    ZeRO-1 outer mode (``sub`` = n > 1): the rank keeps the whole bf16 shard but
    Adam state only for optimizer sub-shard ``node`` of it (``ns / n`` elements)."""

    def __init__(self, lay: StageLayout, D: int, z: int, dev, sub: int = 1, node: int = 0):
        self.lay = lay
        n, ns = lay.numel, lay.shard_numel
        nsub = ns // sub
        self.sub, self.nsub = sub, nsub
        self.gathered = torch.zeros(n, dtype=BF16, device=dev)
        self.shard_bf16 = self.gathered[z * ns:(z + 1) * ns]      # in-place all-gather layout
        sub_i = node if sub > 1 else 0  # DP outer mode: every replica updates its whole shard
        self.sub_bf16 = self.shard_bf16[sub_i * nsub:(sub_i + 1) * nsub]  # AG_PARAM_INTER layout
        self.master = torch.zeros(nsub, dtype=F32, device=dev)
        self.exp_avg = torch.zeros(nsub, dtype=F32, device=dev)
        self.exp_avg_sq = torch.zeros(nsub, dtype=F32, device=dev)
        self.grad_shard = torch.zeros(ns, dtype=F32, device=dev)
        self.grad_sub = self.grad_shard if sub == 1 else torch.zeros(nsub, dtype=F32, device=dev)
        self.grad_full = self.grad_shard if D == 1 else torch.zeros(n, dtype=F32, device=dev)
        self.p: dict = {}
        self.g: dict = {}
        for s in lay.slots:
            key = (s.name, s.layer)
            self.p[key] = self.gathered[s.offset:s.offset + s.numel].view(*s.shape)
            self.g[key] = self.grad_full[s.offset:s.offset + s.numel].view(*s.shape)
        self.ag_event = None        # compute must wait before using gathered params
        self.opt_ready = None       # this stage's shard is updated (early optimizer); AG waits here
        self.grad_free_event = None  # compute must wait before writing grad_full again
        # Gradients are never memset: the first writer of each tensor in an accumulation
        # window (a step at D == 1, one unit's reduce-scatter at D > 1) stores instead of
        # accumulating.  Only the embedding grads (row scatter-add) are zeroed.
        self.scatter_keys = [k for k in self.g if k[0] in ("wte", "wpe")]
        self.new_window()
        self.chunks = opt_chunks(lay)

    def opt_slice(self, key):
        """(lo, hi) element range of optimizer chunk ``key`` ("embed", "head" or a layer)."""
        return self.chunks[key]

    def new_window(self) -> None:
        self.fresh = set(self.g).difference(self.scatter_keys)

    def accumulate(self, key) -> bool:
        """False exactly once per window for ``key``: that writer overwrites."""
        if key in self.fresh:
            self.fresh.discard(key)
            return False
        return True

    def zero_scatter_grads(self, stream) -> None:
        for k in self.scatter_keys:
            ops.zero(self.g[k], stream=stream)


class Runtime:
    """Everything one rank needs to execute ZeroPP steps for a fixed config."""

    def __init__(self, spec: GPTSpec, model: ModelSpec, cfg: ParallelConfig, placement: Placement,
                 sched: Schedule, rank: int = 0, world: int = 1, device: int | None = None,
                 timeline: bool = False, early_opt: bool | None = None, cuda_graph: bool = False,
                 aux_stream: bool = True, host_trace: bool = False, memory_check: bool = True,
                 rs_wire: str = "bf16", stream_priority: bool = False, nccl_max_channels: int | None = 8,
                 overlap_tail: bool = True):
        """``early_opt``: None = auto (on when D > 1, see below); ``cuda_graph``: replay the
        task list as a CUDA graph (one rank); ``aux_stream``: bias / norm-parameter column
        reductions on a side stream; ``host_trace``: print each task as it is enqueued
        (first two steps, debugging); ``memory_check``: refuse configurations whose estimated
        peak does not fit (see below); ``nccl_max_channels``: cap on the CTAs (channels) an NCCL
        collective may occupy -- NCCL's default takes SMs the concurrent GEMMs need (N=4 P2 x D2:
        8 channels +4.0% tokens/s vs the default, profiles/r02/nccl_channels_ab.txt; None keeps
        NCCL's choice; an NCCL_MAX_NCHANNELS already in the environment wins); ``rs_wire``: "bf16" (the reference's byte model,
        `schedules.py:76-78`) or "fp32" (RS_GRAD sums in fp32 on the wire: twice the bytes, no
        bf16 rounding of the partial sums -- tools/rs_wire_drift.py measures the difference);
        ``overlap_tail``: with the early optimizer, the step's last reduce-scatters and AdamW
        run on their side streams into the next step's first forward tasks instead of holding
        the compute stream at OPT (see ``_optimizer``)."""
        self.nccl_max_channels = nccl_max_channels
        if rs_wire not in ("bf16", "fp32"):
            raise ValueError("rs_wire must be 'bf16' or 'fp32'")
        self.rs_wire = rs_wire
        if world != cfg.pp_size * cfg.dp_size * cfg.inter_node_dp:
            raise ValueError(f"world size {world} != n*P*D = "
                             f"{cfg.inter_node_dp * cfg.pp_size * cfg.dp_size}")
        if model.num_layers != spec.num_layers or model.hidden_size != spec.hidden or \
                model.seq_len != spec.seq_len:
            raise ValueError("ModelSpec and GPTSpec disagree on L / h / s")
        if cfg.microbatch_samples != spec.microbatch_samples:
            raise ValueError("ParallelConfig.microbatch_samples != GPTSpec.microbatch_samples")
        bad = validate(sched, placement, cfg)
        if bad:
            raise ValueError(f"schedule failed validation: {bad[0]}")
        self.spec, self.model, self.cfg, self.pl, self.sched = spec, model, cfg, placement, sched
        self.rank, self.world = rank, world
        self.P, self.D, self.n = cfg.pp_size, cfg.dp_size, cfg.inter_node_dp
        self.node, self.p, self.z = rank_coords(rank, self.n, self.P, self.D)
        self.dp_index = self.node * self.D + self.z     # which slice of the global batch
        self.sub = optimizer_sub(cfg)
        self.S = cfg.num_stages
        self.timeline = timeline
        if device is None:
            device = torch.cuda.current_device()
        self.dev = torch.device("cuda", device)
        torch.cuda.set_device(self.dev)
        if memory_check:
            # A configuration that overfills HBM does not fail cleanly here: the caching
            # allocator's release-and-retry path calls cudaFree, a device-wide synchronisation,
            # while NCCL kernels spin on peers -- the job hangs (seen with P2 x D2 B16 U16).
            static, act = memory_estimate(spec, model, cfg, placement, sched, self.p)
            total = torch.cuda.get_device_properties(self.dev).total_memory
            if static + act + 10e9 > total:
                raise MemoryError(
                    f"rank {rank}: estimated peak {static / 1e9:.1f} GB static + {act / 1e9:.1f} GB activations "
                    f"(+10 GB margin) exceeds {total / 1e9:.1f} GB; lower U or microbatch_samples, or raise P / D")
        lib.load()
        lib.call("zpp_preload_kernels")  # no lazy kernel loading once NCCL kernels can spin
        self.tasks = list(sched.per_device[self.p])
        self.local_stages = placement.device_stages(self.p)
        self.stages: dict[int, _Stage] = {}
        for s in self.local_stages:
            lay = stage_layout(spec, s, self.S, placement.stage_to_layers[s], self.D, self.sub)
            self.stages[s] = _Stage(lay, self.D, self.z, self.dev, self.sub, self.node)
        # stream_priority=True: the critical path (compute, collectives, P2P) gets the highest
        # stream priority, the side streams (aux column reductions, early AdamW) the lowest, so
        # the block scheduler fills freed SMs from the critical path first.  Off by default:
        # neutral to -0.4% at N=1 (tools/step_ab.py, profiles/r02/step_ab_priority.txt).
        hi = torch.cuda.Stream.priority_range()[1] if stream_priority else 0
        mk = lambda prio=hi: torch.cuda.Stream(device=self.dev, priority=prio)  # noqa: E731
        self.s_comp, self.s_ag, self.s_rs = mk(), mk(), mk()
        self.s_act_send, self.s_act_recv, self.s_grad_send, self.s_grad_recv = mk(), mk(), mk(), mk()
        # parameter-gradient column reductions (bias, norm gamma / beta) only feed RS / OPT:
        # they run on this side stream beside the next GEMMs (aux_stream=False keeps them inline)
        self.s_aux = mk(0) if aux_stream else self.s_comp
        # Early optimizer: a stage's AdamW starts on its own stream as soon as the stage's
        # gradients are final (its last W at D == 1, layer by layer; its last RS_GRAD at
        # D > 1), overlapping the remaining B / W work instead of trailing the step.  The OPT
        # task still orders everything after it (early_opt=False: OPT runs it all).
        # Default on at D > 1, where it lets the next step's AG_PARAM of a stage start early;
        # at D == 1 there is nothing to overlap but the GEMMs, which under the power cap only
        # slows them (measured: profiles/r01c_ab_n1_aux_earlyopt_b2.txt), so it is off there.
        self.early_opt = self.n == 1 and (self.D > 1 if early_opt is None else bool(early_opt))
        self.overlap_tail = bool(overlap_tail)
        self.s_opt = mk(0)
        # CUDA-graph mode (cuda_graph=True; one rank, no early optimizer): the task list up to
        # OPT is captured once, on the second step, and replayed; OPT runs eagerly after it
        # (AdamW's bias correction depends on the step number).  Shapes, buffers and the task
        # order are static, so a replay is the same launches without the host in the loop.
        self.graph_mode = bool(cuda_graph) and world == 1 and cfg.inter_node_dp == 1
        self.host_trace = host_trace
        self._graph = None
        self._final_w, self._final_rs = {}, {}
        for i, t in enumerate(self.tasks):
            if t.kind is TaskKind.W:
                self._final_w[t.stage] = i
            elif t.kind is TaskKind.RS_GRAD:
                self._final_rs[t.stage] = i
        T, h = spec.tokens_per_microbatch, spec.hidden
        # column-reduction workspaces carry re-armed tickets: zero them once
        self.ln_ws = torch.zeros(ops.layernorm_bwd_workspace(T, h), dtype=F32, device=self.dev)
        self.cs_ws = torch.zeros(ops.colsum_workspace(T, 4 * h), dtype=F32, device=self.dev)
        self.attn_ws = torch.empty(ops.attn_bwd_workspace(spec.microbatch_samples, spec.seq_len,
                                                          spec.heads, spec.head_dim),
                                   dtype=F32, device=self.dev)
        max_n = max(st.lay.numel for st in self.stages.values())
        max_ns = max(st.lay.shard_numel for st in self.stages.values())
        if self.D > 1 or self.n > 1:
            self.rs_send = torch.empty(max_n, dtype=BF16, device=self.dev)
            self.rs_recv = torch.empty(max_ns, dtype=BF16, device=self.dev)
            if self.rs_wire == "fp32" and self.D > 1:  # intra-group RS sums fp32 grad_full directly
                self.rs_recv32 = torch.empty(max_ns, dtype=F32, device=self.dev)
        self.loss_sum = torch.zeros(1, dtype=F32, device=self.dev)
        self.step_count = 0
        self.opt_event = None
        self.comms: dict = {}
        if world > 1:
            self._init_comms()
        self.init_params()

    # ------------------------------------------------------------------ setup
    def _init_comms(self) -> None:
        """Create ZeRO, P2P and outer communicators in one global order (no init deadlock).
        Keys are node-local; a rank only joins the communicators of its own node, plus
        ("inter",) = its (p, z) peers in the other n - 1 replicas."""
        import torch.distributed as dist
        if self.nccl_max_channels:
            os.environ.setdefault("NCCL_MAX_NCHANNELS", str(self.nccl_max_channels))  # read at NCCL init
        lib.load_nccl()
        plan = comm_plan(self.n, self.P, self.D)
        import ctypes
        uids = []
        if self.rank == 0:
            for _ in plan:
                b = ctypes.create_string_buffer(128)
                lib.call("zpp_nccl_unique_id", b)
                uids.append(b.raw)
        obj = [uids]
        dist.broadcast_object_list(obj, src=0)
        uids = obj[0]
        for (key, ranks), uid in zip(plan, uids):
            if self.rank in ranks:
                handle = ctypes.c_void_p()
                lib.call("zpp_comm_init", uid, len(ranks), ranks.index(self.rank), ctypes.byref(handle))
                self.comms[key] = handle

    def init_params(self) -> None:
        """Deterministic init of this rank's shards (identical for every n x P x D split)."""
        with torch.cuda.stream(self.s_comp):
            for st in self.stages.values():
                full = st.master if st.sub == 1 else torch.empty(st.lay.shard_numel, dtype=F32, device=self.dev)
                for slot, t0, s0, cnt in shard_init_ranges(st.lay, self.z):
                    ops.init_param(full[s0:s0 + cnt], st.shard_bf16[s0:s0 + cnt], self.spec.seed,
                                   init_offset(slot.uid) + t0, slot.mean, slot.std, stream=self.s_comp)
                if st.sub > 1:
                    st.master.copy_(full[self.node * st.nsub:(self.node + 1) * st.nsub])
                    full.record_stream(self.s_comp)
        self.opt_event = self._record(self.s_comp)
        if self.D == 1:
            for st in self.stages.values():
                st.ag_event = None

    # ------------------------------------------------------------------ helpers
    @staticmethod
    def _record(stream, timing: bool = False):
        ev = torch.cuda.Event(enable_timing=timing)
        ev.record(stream)
        return ev

    def _wait(self, ev, kind: str | None = None):
        """Make the compute stream wait on ``ev``; measure the stall if timing."""
        if ev is None:
            return
        if self.timeline and kind is not None:
            e0 = self._record(self.s_comp, True)
            self.s_comp.wait_event(ev)
            e1 = self._record(self.s_comp, True)
            self._waits.append((kind, e0, e1, self.tasks[self._ti].task_id))
            self._task_start = e1  # the task's own work starts after its last wait
        else:
            self.s_comp.wait_event(ev)

    def _begin(self, stream) -> None:
        """Mark where a side-stream task's own work starts (after its stream waits)."""
        if self.timeline:
            self._task_start = self._record(stream, True)

    def _dev_of(self, s: int) -> int:
        return self.pl.stage_to_device[s]

    def _peer_rank(self, p: int) -> int:
        return p * self.D + self.z

    # ------------------------------------------------------------------ step
    def step(self, ids: torch.Tensor, labels: torch.Tensor) -> StepResult:
        """Execute one step.  ``ids`` / ``labels``: contiguous int64 [B, b*s] device
        tensors holding this ZeRO rank's micro-batches (labels = next tokens)."""
        spec, cfg = self.spec, self.cfg
        B, b, s_len = cfg.microbatches, spec.microbatch_samples, spec.seq_len
        assert ids.shape == (B, b * s_len) and labels.shape == (B, b * s_len)
        self._ids, self._labels = ids, labels
        self.nccl_bytes = {"intra": 0, "inter": 0}
        self._stash: dict = {}
        self._local_act: dict = {}
        self._local_grad: dict = {}
        self._waits: list = []
        self._rs_events: list = []
        self._grad_scale = 1.0 / (self.n * self.D * B * b * s_len)
        self.step_count += 1
        if self.graph_mode and not self.early_opt and self.step_count >= 2 and self.tasks[-1].kind is TaskKind.OPT:
            return self._graph_step(ids, labels)
        times = {}
        comp = self.s_comp
        comp.wait_stream(torch.cuda.current_stream(self.dev))
        t_start = self._record(comp, True)
        trace = self.host_trace and self.step_count <= 2
        with torch.cuda.stream(comp):
            ops.zero(self.loss_sum, stream=comp)
            self._opt_done: set = set()
            self._opt_ev = None
            for ti, task in enumerate(self.tasks):
                self._ti = ti
                if trace:
                    print(f"[r{self.rank} {time.perf_counter():.3f}] {task.task_id} "
                          f"alloc={torch.cuda.memory_allocated(self.dev) / 1e9:.1f}G "
                          f"reserved={torch.cuda.memory_reserved(self.dev) / 1e9:.1f}G", flush=True)
                stream = self._stream_of(task)
                e0 = self._record(stream, True) if self.timeline else None
                self._task_start = None
                self._run(task)
                if self.timeline:
                    times[task] = (self._task_start or e0, self._record(stream, True))
        t_end = self._record(comp, True)
        torch.cuda.current_stream(self.dev).wait_stream(comp)
        self._t = (t_start, t_end, times)
        tokens_done = B * b * s_len if (self.S - 1) in self.stages else 0
        return StepResult(self.loss_sum, tokens_done, nccl_bytes_intra=self.nccl_bytes["intra"],
                          nccl_bytes_inter=self.nccl_bytes["inter"])

    def _graph_step(self, ids: torch.Tensor, labels: torch.Tensor) -> StepResult:
        comp = self.s_comp
        n_graph = len(self.tasks) - 1  # everything but the trailing OPT
        if self._graph is None:
            self._g_ids, self._g_labels = ids, labels  # the graph reads these buffers
            import gc
            gc.collect()
            torch.cuda.synchronize(self.dev)
            torch.cuda.empty_cache()  # the eager steps' cached blocks would double the peak
            saved = (ops.PROFILE.active, ops.PROFILE.time_gemms, ops.PROFILE.launches)
            ops.PROFILE.active, ops.PROFILE.time_gemms, ops.PROFILE.launches = True, False, 0
            timeline, self.timeline = self.timeline, False
            g = torch.cuda.CUDAGraph()
            try:
                with torch.cuda.graph(g, stream=comp):
                    ops.zero(self.loss_sum, stream=comp)
                    self._opt_done, self._opt_ev = set(), None
                    for ti in range(n_graph):
                        self._ti = ti
                        self._run(self.tasks[ti])
                    self._join_aux(comp)
            finally:
                self.timeline = timeline
                self._graph_launches = ops.PROFILE.launches
                ops.PROFILE.active, ops.PROFILE.time_gemms, ops.PROFILE.launches = saved
            self._graph = g
        else:
            if ids.data_ptr() != self._g_ids.data_ptr():
                self._g_ids.copy_(ids)
            if labels.data_ptr() != self._g_labels.data_ptr():
                self._g_labels.copy_(labels)
            self._ids, self._labels = self._g_ids, self._g_labels
        comp.wait_stream(torch.cuda.current_stream(self.dev))
        t_start = self._record(comp, True)
        with torch.cuda.stream(comp):
            self._graph.replay()
            ops._count(self._graph_launches)
            self._opt_done, self._opt_ev = set(), None
            for ti in range(n_graph, len(self.tasks)):
                self._ti = ti
                self._run(self.tasks[ti])
        t_end = self._record(comp, True)
        torch.cuda.current_stream(self.dev).wait_stream(comp)
        self._t = (t_start, t_end, {})
        spec, cfg = self.spec, self.cfg
        tokens_done = cfg.microbatches * spec.tokens_per_microbatch if (self.S - 1) in self.stages else 0
        return StepResult(self.loss_sum, tokens_done, nccl_bytes_intra=self.nccl_bytes["intra"],
                          nccl_bytes_inter=self.nccl_bytes["inter"])

    def join(self, stream=None) -> None:
        """Order ``stream`` (default: the current stream) after all work this runtime has
        enqueued on any of its streams -- including an overlapped step tail."""
        stream = stream or torch.cuda.current_stream(self.dev)
        for st in (self.s_comp, self.s_ag, self.s_rs, self.s_aux, self.s_opt, self.s_act_send, self.s_act_recv,
                   self.s_grad_send, self.s_grad_recv):
            if st is not stream:
                stream.wait_stream(st)

    def finish_timing(self, res: StepResult) -> StepResult:
        """Resolve CUDA-event timings of the last step.  With a timeline this synchronizes the
        device (every task's events); without one only the compute stream's end of step, so an
        overlapped tail (``overlap_tail``) keeps running into the next step -- call
        :meth:`join` or ``torch.cuda.synchronize()`` before reading parameters directly."""
        t_start, t_end, times = self._t
        if self.timeline:
            torch.cuda.synchronize(self.dev)
        else:
            t_end.synchronize()
        res.step_ms = t_start.elapsed_time(t_end)
        if self.timeline:
            res.task_times = {t: (t_start.elapsed_time(a), t_start.elapsed_time(b)) for t, (a, b) in times.items()}
            res.busy_ms = sum(e - s for t, (s, e) in res.task_times.items() if t.is_compute)
            res.waits = [(k, tid, a.elapsed_time(b)) for k, a, b, tid in self._waits]
            res.exposed_comm_ms = sum(ms for k, _, ms in res.waits if k == "zero")
            res.p2p_wait_ms = sum(ms for k, _, ms in res.waits if k == "p2p")
        return res

    def _stream_of(self, task: Task):
        if task.kind in (TaskKind.AG_PARAM, TaskKind.AG_PARAM_INTER):
            return self.s_ag
        if task.kind in (TaskKind.RS_GRAD, TaskKind.AR_GRAD, TaskKind.RS_GRAD_INTER):
            return self.s_rs
        return self.s_comp

    def _run(self, task: Task) -> None:
        k = task.kind
        if k is TaskKind.F:
            self._forward(task.stage, task.microbatch)
        elif k is TaskKind.B:
            self._backward_input(task.stage, task.microbatch)
        elif k is TaskKind.W:
            self._backward_weight(task.stage, task.microbatch)
        elif k is TaskKind.R:
            self._recompute(task.stage, task.microbatch)
        elif k is TaskKind.AG_PARAM:
            self._all_gather(task.stage)
        elif k is TaskKind.RS_GRAD:
            self._reduce_scatter(task.stage)
        elif k is TaskKind.OPT:
            self._optimizer()
        elif k is TaskKind.AR_GRAD:
            self._outer_grad(reduce_scatter=False)
        elif k is TaskKind.RS_GRAD_INTER:
            self._outer_grad(reduce_scatter=True)
        elif k is TaskKind.AG_PARAM_INTER:
            self._outer_gather()
        else:
            raise NotImplementedError(f"task kind {k}")

    # ------------------------------------------------------------------ comm tasks
    def _all_gather(self, s: int) -> None:
        st = self.stages[s]
        if self.D == 1:
            return  # nothing moves; the previous AG_PARAM_INTER's event (if any) stays armed
        # shards are final once the previous OPT ran -- for an early-optimized stage, once
        # its own AdamW ran (the gather then overlaps the previous step's remaining work)
        self.s_ag.wait_event(st.opt_ready if st.opt_ready is not None else self.opt_event)
        self._begin(self.s_ag)
        ns = st.lay.shard_numel
        lib.call("zpp_allgather", self.comms[("ag", self.p)], st.shard_bf16.data_ptr(),
                 st.gathered.data_ptr(), ns, 0, self.s_ag.cuda_stream)
        self.nccl_bytes["intra"] += (self.D - 1) * ns * 2
        st.ag_event = self._record(self.s_ag)

    def _reduce_scatter(self, s: int) -> None:
        st = self.stages[s]
        if self.D == 1:
            return  # the stage grad IS the shard grad; nothing moves (0 bytes)
        rs = self.s_rs
        rs.wait_event(self._record(self.s_comp))   # all B/W of (s, u) enqueued before this point
        self._join_aux(rs)                           # ... and their parameter-grad reductions
        self._begin(rs)
        n, ns = st.lay.numel, st.lay.shard_numel
        if st.opt_ready is not None:
            rs.wait_event(st.opt_ready)  # grad_shard: the previous step's AdamW read and zeroed it
        if self.rs_wire == "fp32":  # the fp32 stage grad IS the send buffer: reduce, then release it
            recv = self.rs_recv32[:ns]
            lib.call("zpp_reduce_scatter", self.comms[("rs", self.p)], st.grad_full.data_ptr(), recv.data_ptr(), ns,
                     1, rs.cuda_stream)
            self.nccl_bytes["intra"] += (self.D - 1) * ns * 4
            st.zero_scatter_grads(rs)
            st.new_window()
            st.grad_free_event = self._record(rs)
            ops.accum_f32(recv, st.grad_shard, stream=rs)
        else:
            send, recv = self.rs_send[:n], self.rs_recv[:ns]
            ops.cast_scale(st.grad_full, send, 1.0, stream=rs)
            st.zero_scatter_grads(rs)
            st.new_window()
            st.grad_free_event = self._record(rs)
            lib.call("zpp_reduce_scatter", self.comms[("rs", self.p)], send.data_ptr(), recv.data_ptr(), ns, 0,
                     rs.cuda_stream)
            self.nccl_bytes["intra"] += (self.D - 1) * ns * 2
            ops.accum(recv, st.grad_shard, stream=rs)
        ev = self._record(rs)
        self._rs_events.append(ev)
        if self.early_opt and self._final_rs.get(s) == self._ti:
            self._early_opt(st, None, [ev])  # this stage's shard grad is final
            self._opt_done.add(s)

    def _outer_grad(self, reduce_scatter: bool) -> None:
        """AR_GRAD (DP outer, `schedules.py:80-81`) or RS_GRAD_INTER (ZeRO-1 outer,
        `:83-84`): the fp32 shard grads of every local stage summed over the n replicas
        holding the same (p, z) shard, on a bf16 wire (the bytes the reference models).
        AR leaves the sum in ``grad_shard``; RS leaves sub-shard ``node`` in ``grad_sub``."""
        if self.n == 1:
            return  # 0-byte task (ZeRO-1 mode on one node)
        rs = self.s_rs
        rs.wait_event(self._record(self.s_comp))  # D == 1: W wrote grad_shard on compute
        self._join_aux(rs)
        self._begin(rs)
        comm = self.comms[("inter",)]
        for st in self.stages.values():
            ns, nsub = st.lay.shard_numel, st.nsub
            wire = self.rs_send[:ns]
            ops.cast_scale(st.grad_shard, wire, 1.0, stream=rs)
            if reduce_scatter:
                recv = self.rs_recv[:nsub]
                lib.call("zpp_reduce_scatter", comm, wire.data_ptr(), recv.data_ptr(), nsub, 0, rs.cuda_stream)
                self.nccl_bytes["inter"] += (self.n - 1) * nsub * 2
                ops.accum(recv, st.grad_sub, stream=rs)   # grad_sub is zero between steps
            else:
                lib.call("zpp_allreduce", comm, wire.data_ptr(), wire.data_ptr(), ns, 0, rs.cuda_stream)
                self.nccl_bytes["inter"] += 2 * (self.n - 1) * ns * 2 // self.n
                ops.zero(st.grad_shard, stream=rs)
                ops.accum(wire, st.grad_shard, stream=rs)
        self._rs_events.append(self._record(rs))

    def _outer_gather(self) -> None:
        """AG_PARAM_INTER (`schedules.py:86-87`): every replica's updated bf16 sub-shard
        -> the full bf16 shard (in place); the next use of the params waits for it."""
        if self.n == 1:
            return
        ag = self.s_ag
        ag.wait_event(self.opt_event)
        self._begin(ag)
        comm = self.comms[("inter",)]
        for st in self.stages.values():
            lib.call("zpp_allgather", comm, st.sub_bf16.data_ptr(), st.shard_bf16.data_ptr(), st.nsub, 0,
                     ag.cuda_stream)
            self.nccl_bytes["inter"] += (self.n - 1) * st.nsub * 2
        ev = self._record(ag)
        self.opt_event = ev            # AG_PARAM of the next step gathers the updated shard
        if self.D == 1:
            for st in self.stages.values():
                st.ag_event = ev       # no AG_PARAM event to wait on: first use waits here

    def _adamw(self, st: _Stage, lo: int, hi: int, stream) -> None:
        spec = self.spec
        ops.adamw(st.master[lo:hi], st.exp_avg[lo:hi], st.exp_avg_sq[lo:hi], st.grad_sub[lo:hi],
                  st.sub_bf16[lo:hi], spec.lr, spec.beta1, spec.beta2, spec.adam_eps, spec.weight_decay,
                  self.step_count, stream=stream)

    def _early_opt(self, st: _Stage, key, after) -> None:
        """AdamW of optimizer chunk ``key`` (None = the whole shard) on the opt stream,
        ordered after the events ``after`` (the chunk's last gradient writers)."""
        for ev in after:
            self.s_opt.wait_event(ev)
        lo, hi = (0, st.nsub) if key is None else st.opt_slice(key)
        self._adamw(st, lo, hi, self.s_opt)
        if self._tail_overlaps():
            ops.zero(st.grad_shard, stream=self.s_opt)  # the next step's reduce-scatters accumulate here
        self._opt_ev = st.opt_ready = self._record(self.s_opt)

    def _tail_overlaps(self) -> bool:
        """Early optimizer at D > 1 (whole-stage AdamW after each stage's last RS_GRAD) with
        every local stage covered: OPT then has nothing left to run on the compute stream."""
        return (self.overlap_tail and self.early_opt and self.D > 1 and self.sub == 1 and not self.capture_grads
                and not self.graph_mode and all(s in self._final_rs for s in self.stages))

    def _optimizer(self) -> None:
        if self._tail_overlaps() and self._opt_done.issuperset(self.stages):
            # Every stage's AdamW is already queued on the opt stream behind its last
            # reduce-scatter, and zeroes its grad_shard there.  Nothing on the compute stream
            # depends on them: the next step's AG_PARAM of a stage waits for that stage's AdamW
            # (opt_ready), its first RS_GRAD for the zeroed grad_shard, its first W for the
            # released grad_full (grad_free_event).  So the tail overlaps the next step's first
            # forward tasks instead of stalling the compute stream here.  Runtime.join() orders
            # a caller's stream after everything (bench.py's timed region ends with it).
            self.opt_event = self._record(self.s_comp)
            return
        for ev in self._rs_events:
            self._wait(ev, "zero")
        self._join_aux(self.s_comp)  # D == 1: bias / norm grads reduced on aux feed this update
        if self._opt_ev is not None:
            self.s_comp.wait_event(self._opt_ev)  # early chunks (overlapped with B / W) done
        for s, st in self.stages.items():
            if s not in self._opt_done:
                self._adamw(st, 0, st.nsub, self.s_comp)
                st.opt_ready = None
        if self.capture_grads:
            self.captured = {s: st.grad_sub.clone() for s, st in self.stages.items()}
        for st in self.stages.values():
            if st.sub > 1:
                ops.zero(st.grad_sub, stream=self.s_comp)    # inter reduce-scatter accumulates here
            if self.D > 1:
                ops.zero(st.grad_shard, stream=self.s_comp)  # reduce-scatter results accumulate here
            else:
                st.zero_scatter_grads(self.s_comp)
                st.new_window()
        self.opt_event = self._record(self.s_comp)

    capture_grads = False
    captured: dict = {}

    def _use_params(self, st: _Stage) -> None:
        if st.ag_event is not None:
            self._wait(st.ag_event, "zero")
            st.ag_event = None

    def _touch_grads(self, st: _Stage) -> None:
        if st.grad_free_event is not None:
            self._wait(st.grad_free_event, "zero")
            st.grad_free_event = None

    # P2P ---------------------------------------------------------------------
    def _send(self, kind: str, t: torch.Tensor, to_p: int) -> None:
        stream = self.s_act_send if kind == "act" else self.s_grad_send
        stream.wait_event(self._record(self.s_comp))
        lib.call("zpp_send", self.comms[(kind, self.p, to_p, self.z)], t.data_ptr(), t.numel(), 0, 1,
                 stream.cuda_stream)
        t.record_stream(stream)

    def _recv(self, kind: str, shape, from_p: int) -> torch.Tensor:
        stream = self.s_act_recv if kind == "act" else self.s_grad_recv
        with torch.cuda.stream(stream):
            buf = torch.empty(*shape, dtype=BF16, device=self.dev)
        lib.call("zpp_recv", self.comms[(kind, from_p, self.p, self.z)], buf.data_ptr(), buf.numel(), 0, 0,
                 stream.cuda_stream)
        self._wait(self._record(stream), "p2p")
        buf.record_stream(self.s_comp)
        return buf

    # ------------------------------------------------------------------ stage math
    def _recomputed(self, s: int) -> bool:
        """Stages whose activations are recomputed by an R task (schedules.py:454-474)."""
        P, V = self.P, self.cfg.stages_per_device
        return self.cfg.recompute is RecomputeMode.FULL and V > 1 and s // P < V - 1

    def _stage_layers(self, st: "_Stage", x: torch.Tensor):
        """Run the stage's transformer blocks on x; returns (per-layer stash, output)."""
        if self.spec.llama:
            return self._llama_layers(st, x)
        spec = self.spec
        T, h, H, dh = spec.tokens_per_microbatch, spec.hidden, spec.heads, spec.head_dim
        b, sl = spec.microbatch_samples, spec.seq_len
        P = st.p
        e = lambda *shape, dt=BF16: torch.empty(*shape, dtype=dt, device=self.dev)  # noqa: E731
        layers = []
        lo, hi = st.lay.layers
        for l in range(lo, hi):
            xn1, mu1, r1 = e(T, h), e(T, dt=F32), e(T, dt=F32)
            ops.layernorm_fwd(x, P[("ln1_g", l)], P[("ln1_b", l)], xn1, mu1, r1, spec.ln_eps)
            qkv = e(T, 3 * h)
            ops.gemm(xn1, P[("w_qkv", l)], qkv, bias=P[("b_qkv", l)])
            o, lse = e(T, h), e(b, H, sl, dt=F32)
            ops.attn_fwd(qkv, o, lse, b, sl, H, dh)
            x1 = e(T, h)
            ops.gemm(o, P[("w_proj", l)], x1, bias=P[("b_proj", l)], resid=x)
            xn2, mu2, r2 = e(T, h), e(T, dt=F32), e(T, dt=F32)
            ops.layernorm_fwd(x1, P[("ln2_g", l)], P[("ln2_b", l)], xn2, mu2, r2, spec.ln_eps)
            u, g = e(T, 4 * h), e(T, 4 * h)
            ops.gemm(xn2, P[("w_fc1", l)], g, epilogue=ops.EPI_BF16_GELU, bias=P[("b_fc1", l)], aux=u)
            x2 = e(T, h)
            ops.gemm(g, P[("w_fc2", l)], x2, bias=P[("b_fc2", l)], resid=x1)
            layers.append({"x": x, "xn1": xn1, "mu1": mu1, "r1": r1, "qkv": qkv, "o": o, "lse": lse,
                           "x1": x1, "xn2": xn2, "mu2": mu2, "r2": r2, "u": u, "g": g})
            x = x2
        return layers, x

    def _llama_layers(self, st: "_Stage", x: torch.Tensor):
        """LLaMA blocks (RMSNorm, RoPE in place on q/k, SwiGLU; no biases)."""
        spec = self.spec
        T, h, H, dh, f = spec.tokens_per_microbatch, spec.hidden, spec.heads, spec.head_dim, spec.ffn
        b, sl = spec.microbatch_samples, spec.seq_len
        P = st.p
        e = lambda *shape, dt=BF16: torch.empty(*shape, dtype=dt, device=self.dev)  # noqa: E731
        layers = []
        lo, hi = st.lay.layers
        for l in range(lo, hi):
            xn1, r1 = e(T, h), e(T, dt=F32)
            ops.rmsnorm_fwd(x, P[("ln1_g", l)], xn1, r1, spec.ln_eps)
            qkv = e(T, 3 * h)
            ops.gemm(xn1, P[("w_qkv", l)], qkv)
            ops.rope(qkv, sl, H, dh, spec.rope_base)
            o, lse = e(T, h), e(b, H, sl, dt=F32)
            ops.attn_fwd(qkv, o, lse, b, sl, H, dh)
            x1 = e(T, h)
            ops.gemm(o, P[("w_proj", l)], x1, resid=x)
            xn2, r2 = e(T, h), e(T, dt=F32)
            ops.rmsnorm_fwd(x1, P[("ln2_g", l)], xn2, r2, spec.ln_eps)
            gu, a = e(T, 2 * f), e(T, f)
            ops.gemm(xn2, P[("w_fc1", l)], gu)
            ops.swiglu_fwd(gu, a)
            x2 = e(T, h)
            ops.gemm(a, P[("w_fc2", l)], x2, resid=x1)
            layers.append({"x": x, "xn1": xn1, "r1": r1, "qkv": qkv, "o": o, "lse": lse,
                           "x1": x1, "xn2": xn2, "r2": r2, "gu": gu, "a": a})
            x = x2
        return layers, x

    def _aux(self, *hold: torch.Tensor):
        """The side stream, ordered after everything enqueued on compute so far; ``hold``
        tensors are kept alive for it (caching-allocator stream tracking)."""
        if self.s_aux is self.s_comp:
            return self.s_comp
        self.s_aux.wait_event(self._record(self.s_comp))
        for t in hold:
            t.record_stream(self.s_aux)
        return self.s_aux

    def _join_aux(self, stream) -> None:
        if self.s_aux is not self.s_comp:
            stream.wait_event(self._record(self.s_aux))

    def _norm_bwd(self, st: "_Stage", dy, x, mean, rstd, gkey, bkey, dx, dresid=None) -> None:
        """LayerNorm (mean given) / RMSNorm backward: dx on compute, gamma / beta grads on aux."""
        P, G = st.p, st.g
        if mean is None:
            ops.rmsnorm_bwd(dy, x, rstd, P[gkey], dx, None, None, dresid=dresid)
        else:
            ops.layernorm_bwd(dy, x, mean, rstd, P[gkey], dx, None, None, None, dresid=dresid)
        acc = st.accumulate(gkey)
        if bkey is not None:
            acc = acc | st.accumulate(bkey)
        held = (dy, x, rstd) if mean is None else (dy, x, mean, rstd)
        ops.norm_param_grads(dy, x, mean, rstd, G[gkey], G[bkey] if bkey is not None else None, self.ln_ws,
                             accumulate=acc, stream=self._aux(*held))

    def _final_norm(self, st: "_Stage", out: torch.Tensor):
        spec, P = self.spec, st.p
        T, h = out.shape
        xf, rf = torch.empty(T, h, dtype=BF16, device=self.dev), torch.empty(T, dtype=F32, device=self.dev)
        if spec.llama:
            ops.rmsnorm_fwd(out, P[("lnf_g", None)], xf, rf, spec.ln_eps)
            return xf, {"xlast": out, "rf": rf}
        muf = torch.empty(T, dtype=F32, device=self.dev)
        ops.layernorm_fwd(out, P[("lnf_g", None)], P[("lnf_b", None)], xf, muf, rf, spec.ln_eps)
        return xf, {"xlast": out, "muf": muf, "rf": rf}

    def _final_norm_bwd(self, st: "_Stage", stash: dict, dxf: torch.Tensor) -> torch.Tensor:
        dx = torch.empty_like(dxf)
        llama = self.spec.llama
        self._norm_bwd(st, dxf, stash.pop("xlast"), None if llama else stash.pop("muf"), stash.pop("rf"),
                       ("lnf_g", None), None if llama else ("lnf_b", None), dx)
        return dx

    def _forward(self, s: int, m: int) -> None:
        spec = self.spec
        st = self.stages[s]
        self._use_params(st)
        T, h = spec.tokens_per_microbatch, spec.hidden
        P = st.p
        e = lambda *shape, dt=BF16: torch.empty(*shape, dtype=dt, device=self.dev)  # noqa: E731
        if s == 0:
            x = e(T, h)
            ops.embed_fwd(self._ids[m], P[("wte", None)], P.get(("wpe", None)), x, spec.seq_len)
        elif self._dev_of(s - 1) == self.p:
            x = self._local_act.pop((s, m))
        else:
            x = self._recv("act", (T, h), self._dev_of(s - 1))
        layers, out = self._stage_layers(st, x)
        if self._recomputed(s):
            stash = {"x_in": x}  # boundary slab only; R(s, m) rebuilds the rest
            del layers
        else:
            stash = {"layers": layers}
        if s == self.S - 1:
            xf, norm_stash = self._final_norm(st, out)
            logits = e(T, spec.vocab)
            ops.gemm(xf, P[("w_lm", None)], logits)
            ops.xent(logits, self._labels[m], self.loss_sum, self._grad_scale)
            stash.update(norm_stash, xf=xf, dlogits=logits)
        elif self._dev_of(s + 1) == self.p:
            self._local_act[(s + 1, m)] = out
        else:
            self._send("act", out, self._dev_of(s + 1))
        self._stash[(s, m)] = stash

    def _recompute(self, s: int, m: int) -> None:
        """R task: re-run the stage forward from the stashed input (schedules.py:466-472)."""
        st = self.stages[s]
        self._use_params(st)
        stash = self._stash[(s, m)]
        layers, _ = self._stage_layers(st, stash.pop("x_in"))
        stash["layers"] = layers

    def _backward_input(self, s: int, m: int) -> None:
        spec = self.spec
        st = self.stages[s]
        self._use_params(st)
        self._touch_grads(st)
        T, h, H, dh = spec.tokens_per_microbatch, spec.hidden, spec.heads, spec.head_dim
        b, sl = spec.microbatch_samples, spec.seq_len
        P, G = st.p, st.g
        e = lambda *shape, dt=BF16: torch.empty(*shape, dtype=dt, device=self.dev)  # noqa: E731
        stash = self._stash[(s, m)]
        if s == self.S - 1:
            dxf = e(T, h)
            ops.gemm(stash["dlogits"], P[("w_lm", None)], dxf, b_t=True)
            dx = self._final_norm_bwd(st, stash, dxf)
        elif self._dev_of(s + 1) == self.p:
            dx = self._local_grad.pop((s, m))
        else:
            dx = self._recv("grad", (T, h), self._dev_of(s + 1))
        lo, hi = st.lay.layers
        for i, l in reversed(list(enumerate(range(lo, hi)))):
            if spec.llama:
                dx = self._llama_layer_bwd(st, stash["layers"], i, l, dx)
                continue
            a = stash["layers"][i]
            d2 = dx
            du = e(T, 4 * h)
            ops.gemm(d2, P[("w_fc2", l)], du, b_t=True, epilogue=ops.EPI_BF16_DGELU, aux=a["u"])
            dxn2 = e(T, h)
            ops.gemm(du, P[("w_fc1", l)], dxn2, b_t=True)
            dx1 = e(T, h)
            self._norm_bwd(st, dxn2, a["x1"], a["mu2"], a["r2"], ("ln2_g", l), ("ln2_b", l), dx1, dresid=d2)
            do = e(T, h)
            ops.gemm(dx1, P[("w_proj", l)], do, b_t=True)
            dqkv = e(T, 3 * h)
            ops.attn_bwd(a["qkv"], a["o"], a["lse"], do, dqkv, self.attn_ws, b, sl, H, dh)
            dxn1 = e(T, h)
            ops.gemm(dqkv, P[("w_qkv", l)], dxn1, b_t=True)
            dxl = e(T, h)
            self._norm_bwd(st, dxn1, a["x"], a["mu1"], a["r1"], ("ln1_g", l), ("ln1_b", l), dxl, dresid=dx1)
            # keep only what W needs: inputs of the linears and their output grads
            stash["layers"][i] = {"xn1": a["xn1"], "o": a["o"], "xn2": a["xn2"], "g": a["g"],
                                  "d2": d2, "du": du, "dx1": dx1, "dqkv": dqkv}
            dx = dxl
        if s == 0:
            stash["demb"] = dx
        elif self._dev_of(s - 1) == self.p:
            self._local_grad[(s - 1, m)] = dx
        else:
            self._send("grad", dx, self._dev_of(s - 1))

    def _llama_layer_bwd(self, st: "_Stage", layers: list, i: int, l: int, dx: torch.Tensor) -> torch.Tensor:
        """Input-gradient of one LLaMA block; leaves what W needs in ``layers[i]``."""
        spec = self.spec
        T, h, H, dh, f = spec.tokens_per_microbatch, spec.hidden, spec.heads, spec.head_dim, spec.ffn
        b, sl = spec.microbatch_samples, spec.seq_len
        P, G = st.p, st.g
        e = lambda *shape, dt=BF16: torch.empty(*shape, dtype=dt, device=self.dev)  # noqa: E731
        a = layers[i]
        d2 = dx
        da = e(T, f)
        ops.gemm(d2, P[("w_fc2", l)], da, b_t=True)
        dgu = e(T, 2 * f)
        ops.swiglu_bwd(da, a["gu"], dgu)
        dxn2 = e(T, h)
        ops.gemm(dgu, P[("w_fc1", l)], dxn2, b_t=True)
        dx1 = e(T, h)
        self._norm_bwd(st, dxn2, a["x1"], None, a["r2"], ("ln2_g", l), None, dx1, dresid=d2)
        do = e(T, h)
        ops.gemm(dx1, P[("w_proj", l)], do, b_t=True)
        dqkv = e(T, 3 * h)
        ops.attn_bwd(a["qkv"], a["o"], a["lse"], do, dqkv, self.attn_ws, b, sl, H, dh)
        ops.rope(dqkv, sl, H, dh, spec.rope_base, inverse=True)   # d(pre-rotation q, k)
        dxn1 = e(T, h)
        ops.gemm(dqkv, P[("w_qkv", l)], dxn1, b_t=True)
        dxl = e(T, h)
        self._norm_bwd(st, dxn1, a["x"], None, a["r1"], ("ln1_g", l), None, dxl, dresid=dx1)
        layers[i] = {"xn1": a["xn1"], "o": a["o"], "xn2": a["xn2"], "a": a["a"],
                     "d2": d2, "dgu": dgu, "dx1": dx1, "dqkv": dqkv}
        return dxl

    def _backward_weight(self, s: int, m: int) -> None:
        st = self.stages[s]
        self._touch_grads(st)
        G = st.g
        stash = self._stash.pop((s, m))
        lo, hi = st.lay.layers
        linears = ((("d2", "a", "w_fc2", None), ("dgu", "xn2", "w_fc1", None), ("dx1", "o", "w_proj", None),
                    ("dqkv", "xn1", "w_qkv", None)) if self.spec.llama else
                   (("d2", "g", "w_fc2", "b_fc2"), ("du", "xn2", "w_fc1", "b_fc1"),
                    ("dx1", "o", "w_proj", "b_proj"), ("dqkv", "xn1", "w_qkv", "b_qkv")))
        if not self.spec.llama:  # bias grads: column sums of the linears' output grads, on aux
            aux = self._aux(*[stash["layers"][i][dy] for i in range(hi - lo) for dy, _, _, _ in linears])
            for i, l in enumerate(range(lo, hi)):
                a = stash["layers"][i]
                for dy, _, _, bias in linears:
                    ops.colsum_acc(a[dy], G[(bias, l)], self.cs_ws, accumulate=st.accumulate((bias, l)), stream=aux)
        early = self.early_opt and self.D == 1 and self._final_w.get(s) == self._ti
        after = [self._record(self.s_aux)] if early and self.s_aux is not self.s_comp else []

        def chunk_done(key):  # every gradient writer of chunk ``key`` is enqueued
            if early:
                self._early_opt(st, key, after + [self._record(self.s_comp)])
                after.clear()

        if s == self.S - 1:
            ops.gemm(stash["dlogits"], stash["xf"], G[("w_lm", None)], a_t=True, b_t=True,
                     epilogue=ops.EPI_F32_ACC if st.accumulate(("w_lm", None)) else ops.EPI_F32)
            chunk_done("head")
        for i, l in reversed(list(enumerate(range(lo, hi)))):
            a = stash["layers"][i]
            for dy, x, w, bias in linears:
                ops.gemm(a[dy], a[x], G[(w, l)], a_t=True, b_t=True,
                         epilogue=ops.EPI_F32_ACC if st.accumulate((w, l)) else ops.EPI_F32)
            chunk_done(l)
        if s == 0:
            ops.embed_bwd(self._ids[m], stash["demb"], G[("wte", None)], G.get(("wpe", None)),
                          self.spec.seq_len)
            chunk_done("embed")
        if early:
            self._opt_done.add(s)


def execute(sched: Schedule, model: ModelSpec, cfg: ParallelConfig, placement: Placement,
            runtime: Runtime, ids: torch.Tensor, labels: torch.Tensor) -> StepResult:
    """Run one ZeroPP training step of ``sched`` on this rank (the engine's
    ``simulate``, `simulation.py:90`).  Returns a timed :class:`StepResult`; with a
    ``timeline=True`` runtime (which synchronizes the device per step) it also carries the whole-job measured
    :class:`~paper_2402_03791_b200.simulation.SimResult` (``res.sim``, fields readable
    directly: ``res.makespan``, ``res.bubble_ratios``, ``res.loss`` ...) -- a
    collective over all ranks when the job is multi-rank."""
    if sched is not runtime.sched:
        raise ValueError("runtime was built for a different schedule")
    t0 = time.perf_counter()
    res = runtime.step(ids, labels)
    res = runtime.finish_timing(res)
    res.host_s = time.perf_counter() - t0
    if runtime.timeline and res.task_times:  # (a CUDA-graph replay carries no per-task times)
        from .timeline import measured_result
        import torch.distributed as dist
        gather = runtime.world > 1 and dist.is_available() and dist.is_initialized()
        res.sim = measured_result(runtime, res, gather=gather)
    return res
