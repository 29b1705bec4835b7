"""ZeroPP training-step benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl zpp|reference]

Metric (BASELINE.json): tokens/s per box for a GPT-6.2B ZeroPP step, plus MFU and
exposed comm ms/step.  One process per GPU (torchrun for N > 1); weak scaling:
every GPU processes 8 micro-batches x 2048 tokens of GPT-6.2B work per step:

    N=1: P1 x D1, B=8,  U=2, V=1      N=2: P2 x D1, B=16, U=8, V=2
    N=4: P2 x D2, B=16, U=8, V=2      N=8: P2 x D4, B=16, U=8, V=2

value  : tokens/s with inputs resident in HBM, CUDA-event time of K steps, max over ranks
e2e    : same metric through the public API ``execute(...)`` with per-step H2D copy of the
         step's token ids/labels from pinned host memory and a D2H read of the loss
roofline: dominant kernel = the tcgen05 GEMM; achieved = algorithmic GEMM FLOPs of the timed
         steps / summed CUDA-event durations of those GEMM launches (on their stream)
cpu_baseline: the CPU fp32 oracle (oracle/gpt_oracle.py) timed on this host on a bounded
         sample (1 GPT-6.2B layer + LM head, 2048 tokens, fwd+bwd), extrapolated to the full
         model by model FLOPs (labelled ``extrapolated``).
--impl reference: that CPU figure, plus the reference package's own generate / validate /
         simulate timed for this config (baseline/_ref) and a fully measured C1 oracle step
         (see run_reference).
"""

from __future__ import annotations

import argparse
import json
import os

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")  # see zpp_preload_kernels
if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION"):
    os.environ["NCCL_DEBUG"] = "WARN"  # keep stdout to the one JSON line (no "NCCL version" banner)
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tokens/s/box GPT-6.2B ZeroPP at 1/2/4/8 B200; MFU; exposed comm ms/step"
# (P, D, B, U, V, b): b = samples per micro-batch (ParallelConfig.microbatch_samples).  b = 2
# (4096-token micro-batches) measured +10% over b = 1 at N=1 (profiles/r01c_n1_microbatch_size.txt):
# M = 4096 GEMMs waste less per FLOP, which is what counts under the 1000 W cap (DESIGN 5a).
SPLITS = {1: (1, 1, 8, 2, 1, 2), 2: (2, 1, 16, 8, 2, 2), 4: (2, 2, 16, 8, 2, 2), 8: (2, 4, 16, 8, 2, 2)}
# other BASELINE configs (parity cases; measured with --model / --split, not the headline line)
MODELS = {"gpt-6.2b": ("gpt_6p2b", "GPT-6.2B (L32 h4096 a32 s2048 V50304, untied head)"),
          "gpt-1.3b": ("gpt_1p3b", "GPT-1.3B (L24 h2048 a16 s2048 V50304, untied head)"),
          "llama-7b": ("llama_7b", "LLaMA-7B (L32 h4096 a32 s4096 V32000, SwiGLU 11008, RoPE, RMSNorm)"),
          "gpt-13b": ("gpt_13b", "GPT-13B (L40 h5120 a40 s2048 V50304, untied head)")}
PEAK_DENSE_TF = 2250.0


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), d["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def _gemm_traffic():
    """Per-launch DRAM bytes of the GEMM launches of one step, from the committed ncu
    capture summary (tools/gemm_traffic.py -> profiles/gemm_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "gemm_traffic.json")) as f:
            d = json.load(f)
        return d["dram_bytes_per_launch"], d["algorithmic_bytes_per_launch"]
    except Exception:
        return None, None


# --------------------------------------------------------------------------- CPU leg
def cpu_sample(threads: int | None = None) -> dict:
    """Time the CPU fp32 oracle on one bounded sample and extrapolate to GPT-6.2B tokens/s."""
    import torch
    from oracle.gpt_oracle import gpt_forward_loss
    from paper_2402_03791_b200.engine import GPTSpec
    threads = threads or os.cpu_count() or 1
    torch.set_num_threads(threads)
    spec = GPTSpec.gpt_6p2b()
    h, V, s, H = spec.hidden, spec.vocab, spec.seq_len, spec.heads
    g = torch.Generator().manual_seed(0)

    def mk(*shape, std=0.02):
        return (torch.randn(*shape, generator=g) * std).requires_grad_(True)
    p = {("wte", None): mk(V, h), ("wpe", None): mk(s, h), ("lnf_g", None): mk(h, std=1.0),
         ("lnf_b", None): mk(h), ("w_lm", None): mk(V, h)}
    for n, shp in [("ln1_g", (h,)), ("ln1_b", (h,)), ("w_qkv", (3 * h, h)), ("b_qkv", (3 * h,)),
                   ("w_proj", (h, h)), ("b_proj", (h,)), ("ln2_g", (h,)), ("ln2_b", (h,)),
                   ("w_fc1", (4 * h, h)), ("b_fc1", (4 * h,)), ("w_fc2", (h, 4 * h)), ("b_fc2", (h,))]:
        p[(n, 0)] = mk(*shp)
    ids = torch.randint(0, V, (1, s), generator=g)
    lab = torch.randint(0, V, (1, s), generator=g)
    t0 = time.perf_counter()
    gpt_forward_loss(p, ids, lab, layers=1, heads=H).backward()
    dt = time.perf_counter() - t0
    sample_flops = s * (72.0 * h * h + 12.0 * s * h + 6.0 * h * V)
    rate = sample_flops / dt
    return {"value": rate / spec.flops_per_token(), "unit": "tokens/s", "cores": threads, "kind": "port",
            "sample": f"oracle fwd+bwd of 1 GPT-6.2B layer + LM head on 1x2048 tokens in {dt:.2f}s "
                      f"({rate / 1e9:.0f} GFLOP/s fp32), extrapolated to 32 layers by model FLOPs"}


# --------------------------------------------------------------------------- clocks
class Clocks:
    def __init__(self, out_dir: str, device: int = 0):
        self.path = os.path.join(out_dir, "clocks.csv")
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            device = int(vis.split(",")[device])
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict | None:
        if self.proc is None:
            return None
        self.proc.terminate()
        self.proc.wait()
        sm, pw, mx, reasons = [], [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
                pw.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        loaded = [i for i, x in enumerate(sm) if x > 0.5 * mx] or list(range(len(sm)))
        return {"sm_mhz": statistics.median(sm[i] for i in loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "power_w": statistics.median(pw[i] for i in loaded) if len(pw) == len(sm) else None}


# --------------------------------------------------------------------------- GPU leg
def run_zpp(args) -> None:
    import torch
    import torch.distributed as dist
    from paper_2402_03791_b200.engine.data import synthetic_tokens as make_tokens
    from paper_2402_03791_b200 import ModelSpec, ParallelConfig, generate, make_placement
    from paper_2402_03791_b200.engine import GPTSpec, Runtime, execute, ops

    N = args.gpus
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != N:
        raise SystemExit(f"--gpus {N} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    P, D, B, U, V, mbs = _split(args)
    spec = getattr(GPTSpec, MODELS[args.model][0])(microbatch_samples=mbs)
    model = ModelSpec(num_layers=spec.num_layers, hidden_size=spec.hidden, seq_len=spec.seq_len)
    cfg = ParallelConfig(pp_size=P, dp_size=D, microbatches=B, unit_size=U, stages_per_device=V,
                         microbatch_samples=mbs)
    pl = make_placement(cfg, model)
    sched = generate(model, cfg, pl)
    import ast
    rt_kw = {k: ast.literal_eval(v) for k, v in (kv.split("=") for kv in args.rt.split(",") if kv)}
    rt = Runtime(spec, model, cfg, pl, sched, rank=rank, world=world, timeline=True, **rt_kw)
    z = rt.z
    # NB distinct synthetic batches, cycled step by step: a repeated batch would be memorised
    # within a few steps (loss -> 0), which is not a training workload
    NB = 4
    toks = make_tokens(NB, D, B, mbs, spec.seq_len, spec.vocab)
    ids_hs = [toks[k, z, :, :, :-1].reshape(B, -1).contiguous().pin_memory() for k in range(NB)]
    lab_hs = [toks[k, z, :, :, 1:].reshape(B, -1).contiguous().pin_memory() for k in range(NB)]
    ids_ds, lab_ds = [x.cuda() for x in ids_hs], [x.cuda() for x in lab_hs]
    ids_h, lab_h = ids_hs[0], lab_hs[0]
    ids_d, lab_d = ids_h.cuda(), lab_h.cuda()
    tokens_per_step = D * B * spec.tokens_per_microbatch

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    # warm-up (also lets the caching allocator settle)
    for k in range(args.warmup):
        rt.step(ids_ds[k % NB], lab_ds[k % NB])
    barrier()

    # ---- kernel-resident timed region (value) ----------------------------------
    clocks = Clocks(args.out_dir, local) if rank == 0 else None
    comp = rt.s_comp
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ops.PROFILE.start(time_gemms=False)  # launch counting only: no per-kernel events here
    barrier()
    ev0.record(comp)
    results = []
    t_host = time.perf_counter()
    for k in range(args.steps):
        results.append(rt.step(ids_ds[k % NB], lab_ds[k % NB]))
    host_ms = (time.perf_counter() - t_host) * 1e3  # enqueue time: the host runs ahead of the GPU
    rt.join(comp)  # the last step's tail (reduce-scatters / AdamW on side streams) is inside the region
    ev1.record(comp)
    barrier()
    launches = ops.PROFILE.launches
    ops.PROFILE.stop()
    dev_ms = max_over_ranks(ev0.elapsed_time(ev1))

    # ---- roofline timed region: same steps, every GEMM bracketed by CUDA events ---
    graph_mode, rt.graph_mode = rt.graph_mode, False  # per-GEMM events need eager launches
    ops.PROFILE.start(time_gemms=True)
    barrier()
    for k in range(args.steps):
        rt.step(ids_ds[k % NB], lab_ds[k % NB])
    barrier()
    gemm_flops, gemm_ms, gemm_calls = ops.PROFILE.stop()
    rt.graph_mode = graph_mode
    clk = clocks.stop() if clocks else None
    # per-step exposed comm from the last step's timeline (max over ranks)
    last = rt.finish_timing(results[-1])
    exposed_ms = max_over_ranks(last.exposed_comm_ms or 0.0)
    p2p_ms = max_over_ranks(last.p2p_wait_ms or 0.0)
    loss = last.loss_sum.item()
    if world > 1:
        lt = torch.tensor([loss])
        dist.all_reduce(lt)
        loss = lt.item()
    loss /= tokens_per_step

    # ---- end-to-end through the public API (host buffers in the timed region) --
    barrier()
    timeline, rt.timeline = rt.timeline, False  # no per-task events: execute() syncs only on the step's end
    t_e2e = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(args.steps):
        ids_d.copy_(ids_hs[k % NB], non_blocking=True)
        lab_d.copy_(lab_hs[k % NB], non_blocking=True)
        r = execute(sched, model, cfg, pl, rt, ids_d, lab_d)
        _ = r.loss_sum.item()
    rt.join()
    e1.record()
    barrier()
    rt.timeline = timeline
    e2e_ms = max_over_ranks(max(e0.elapsed_time(e1), (time.perf_counter() - t_e2e) * 1e3))
    mem_gb = max_over_ranks(torch.cuda.max_memory_allocated() / 1e9)

    if rank == 0:
        burst, sustained, hbm, kind = _peaks()
        step_ms = dev_ms / args.steps
        value = tokens_per_step * args.steps / (dev_ms / 1e3)
        flops_tok = spec.flops_per_token()
        achieved_tf = gemm_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else None
        traffic, alg_bytes = _gemm_traffic()
        line = {
            "metric": METRIC if args.model == "gpt-6.2b" else METRIC.replace("GPT-6.2B", args.model.upper()),
            "value": round(value, 1), "unit": "tokens/s", "n_gpus": N,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded CPU randint tokens, 4 distinct batches cycled; deterministic counter-hash init)",
            "config": {"workload": f"{args.model.upper()} ZeroPP step, P{P} x D{D}, B={B} micro-batches/ZeRO "
                                   f"rank, U={U}, V={V}, b={mbs}, s={spec.seq_len}",
                       "model": MODELS[args.model][1],
                       "global_batch": D * B * mbs, "seq_len": spec.seq_len, "parallelism": f"pp{P}xzero{D}",
                       "tokens_per_step": tokens_per_step,
                       "cuda_graph": rt._graph is not None,
                       "overlap_tail": rt._tail_overlaps(),
                       **({"runtime_overrides": args.rt} if args.rt else {}),
                       "l2": "inputs larger than L2 (each step streams >10 GB of weights/activations)"},
            "mfu": {"vs_2250_dense": round(value * flops_tok / (N * PEAK_DENSE_TF * 1e12), 4),
                    f"vs_{kind}_{sustained}": round(value * flops_tok / (N * sustained * 1e12), 4)},
            "exposed_comm_ms_per_step": round(exposed_ms, 3),
            "host_enqueue_ms_per_step": round(host_ms / args.steps, 1),
            "p2p_wait_ms_per_step": round(p2p_ms, 3),
            "loss": round(loss, 5),
            "max_mem_gb": round(mem_gb, 1),
            "e2e": {"value": round(tokens_per_step * args.steps / (e2e_ms / 1e3), 1), "unit": "tokens/s",
                    "h2d_bytes_per_step": int((ids_h.numel() + lab_h.numel()) * 8 * world),
                    "d2h_bytes_per_step": 4 * world},
            "roofline": {"bound": "tensor", "kernel": "zpp gemm_tcgen05 (all F/B/W linears)",
                         "achieved": round(achieved_tf, 1) if achieved_tf else None, "peak": sustained,
                         "peak_kind": f"{kind} sustained bf16", "unit": "TFLOP/s",
                         "frac": round(achieved_tf / sustained, 4) if achieved_tf else None,
                         "gemm_launches": gemm_calls,
                         "traffic": round(traffic) if traffic else None,
                         "traffic_unit": "DRAM bytes per GEMM launch (ncu, profiles/gemm_traffic.json)",
                         "algorithmic_bytes_per_launch": round(alg_bytes) if alg_bytes else None},
            "gpu_launches": launches,
            "clocks": clk,
        }
        if not args.no_cpu and world == 1:  # the CPU baseline is an N=1 leg (rank 0 only)
            line["cpu_baseline"] = cpu_sample()
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _split(args):
    """(P, D, B, U, V, b) of --gpus, or of --split PxD:B:U:V[:b]; --mb-size overrides b."""
    if not args.split:
        P, D, B, U, V, b = SPLITS[args.gpus]
    else:
        f = args.split.split(":")
        P, D = (int(x) for x in f[0].lower().split("x"))
        B, U, V = int(f[1]), int(f[2]), int(f[3])
        b = int(f[4]) if len(f) > 4 else 1
        if P * D != args.gpus:
            raise SystemExit(f"--split {args.split}: P*D != --gpus {args.gpus}")
    if getattr(args, "mb_size", None):
        b = args.mb_size
    return P, D, B, U, V, b


def reference_schedule_path(args) -> dict:
    """The reference's OWN CPU path for this config, timed here: ``zeroppsim`` generate +
    validate + simulate (`schedules.py:555-567`, `validation.py:99-135`, `simulation.py:90-158`),
    imported read-only from ``baseline/_ref`` (pip-installed from the reference, git-ignored,
    shipped to the GPU box).  Single-threaded pure Python, as the reference runs.  Also checks
    that its schedule is the one this engine executes (same per-device task ids)."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "zeroppsim")):
        return {"unavailable": "baseline/_ref not installed (see DESIGN.md, reference arm)"}
    sys.path.insert(0, ref_dir)
    import zeroppsim as R
    from paper_2402_03791_b200 import ModelSpec, ParallelConfig, generate, make_placement
    from paper_2402_03791_b200.engine import GPTSpec
    P, D, B, U, V, mbs = _split(args)
    spec = getattr(GPTSpec, MODELS[args.model][0])(microbatch_samples=mbs)
    mk = dict(num_layers=spec.num_layers, hidden_size=spec.hidden, seq_len=spec.seq_len)
    pk = dict(pp_size=P, dp_size=D, microbatches=B, unit_size=U, stages_per_device=V, microbatch_samples=mbs)
    m, c = R.ModelSpec(**mk), R.ParallelConfig(**pk)
    pl = R.make_placement(c, m)
    costs = R.CommCostModel(intra_node_bandwidth=900e9, inter_node_bandwidth=50e9)
    reps = 20
    t = {"generate": [], "validate": [], "simulate": []}
    for _ in range(reps):
        t0 = time.perf_counter()
        sched = R.generate(m, c, pl)
        t1 = time.perf_counter()
        bad = R.validate(sched, pl, c)
        t2 = time.perf_counter()
        sim = R.simulate(sched, m, c, pl, costs)
        t3 = time.perf_counter()
        t["generate"].append(t1 - t0)
        t["validate"].append(t2 - t1)
        t["simulate"].append(t3 - t2)
    ours = generate(ModelSpec(**mk), ParallelConfig(**pk), make_placement(ParallelConfig(**pk), ModelSpec(**mk)))
    same = [[x.task_id for x in d] for d in sched.per_device] == [[x.task_id for x in d] for d in ours.per_device]
    out = {f"{k}_ms": round(statistics.median(v) * 1e3, 3) for k, v in t.items()}
    out.update({"cores": 1, "tasks": sched.task_count(), "violations": len(bad), "makespan_units": sim.makespan,
                "same_task_order_as_engine": same, "repeats": reps,
                "source": "zeroppsim 0.1.0 from baseline/_ref (the reference package itself)"})
    return out


def c1_oracle_step(threads: int) -> dict:
    """A MEASURED CPU step of BASELINE config C1 (tiny GPT L4 h256 s128, P2 x D2, B8 U4 V2):
    the fp32 oracle's forward + backward + AdamW over the global batch (2 x 8 x 128 tokens),
    the whole step, nothing extrapolated."""
    import torch
    from oracle.gpt_oracle import make_tokens, oracle_step
    from oracle.init_oracle import init_values
    from paper_2402_03791_b200 import ModelSpec, ParallelConfig, make_placement
    from paper_2402_03791_b200.engine import GPTSpec
    from paper_2402_03791_b200.engine.model import init_offset, stage_layout
    torch.set_num_threads(threads)
    spec = GPTSpec.tiny()
    cfg = ParallelConfig(pp_size=2, dp_size=2, microbatches=8, unit_size=4, stages_per_device=2)
    pl = make_placement(cfg, ModelSpec(num_layers=spec.num_layers, hidden_size=spec.hidden, seq_len=spec.seq_len))
    params = {}
    for st in range(cfg.num_stages):
        for sl in stage_layout(spec, st, cfg.num_stages, pl.stage_to_layers[st], cfg.dp_size).slots:
            params[(sl.name, sl.layer)] = torch.from_numpy(
                init_values(sl.numel, spec.seed, init_offset(sl.uid), sl.mean, sl.std)).view(*sl.shape)
    tok = make_tokens(1, 2, 8, 1, spec.seq_len, spec.vocab)[0]
    ids, labels = tok[..., :-1].reshape(16, -1), tok[..., 1:].reshape(16, -1)
    kw = dict(layers=spec.num_layers, heads=spec.heads, lr=spec.lr)
    oracle_step(params, ids, labels, **kw)  # warm-up
    times = []
    for _ in range(3):
        t0 = time.perf_counter()
        oracle_step(params, ids, labels, **kw)
        times.append(time.perf_counter() - t0)
    dt = statistics.median(times)
    return {"value": round(ids.numel() / dt, 1), "unit": "tokens/s", "ms_per_step": round(dt * 1e3, 2),
            "tokens_per_step": ids.numel(), "cores": threads, "measured": True,
            "config": "C1 tiny GPT L4 h256 s128, global batch 16 x 128 tokens, fwd+bwd+AdamW"}


def run_reference(args) -> None:
    """``--impl reference``: the reference's CPU side of this workload on this host.

    The reference (`zeroppsim`) is a stdlib-only schedule SIMULATOR with no step arithmetic
    (SURVEY.md section 0), so the arm reports three things, each labelled:
    * ``value``: the CPU fp32 oracle port of the GPT-6.2B step on all host cores -- a bounded
      sample per "step" (1 layer + LM head on 2048 tokens), EXTRAPOLATED to the full model by
      model FLOPs (``extrapolated: true``); ``ms_per_step`` = tokens_per_step / value, so the
      line is self-consistent (a full CPU step would take ~this long);
    * ``reference_cpu_path``: the reference's own generate + validate + simulate for this
      config, timed (ms, 1 core), from the reference package itself (baseline/_ref);
    * ``c1_measured_step``: a fully MEASURED fp32 oracle step of BASELINE config C1.
    Rank 0 only; other ranks exit without work."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_sample(threads)
    vals, last = [], None
    for _ in range(args.steps):
        last = cpu_sample(threads)
        vals.append(last["value"])
    value = statistics.median(vals)
    P, D, B, U, V, mbs = _split(args)
    from paper_2402_03791_b200.engine import GPTSpec
    spec = getattr(GPTSpec, MODELS[args.model][0])(microbatch_samples=mbs)
    tokens_per_step = D * B * spec.tokens_per_microbatch
    line = {"metric": METRIC, "impl": "reference", "value": round(value, 3), "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(tokens_per_step / value * 1e3, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
            "extrapolated": True,
            "config": {"workload": f"{args.model.upper()} ZeroPP step, P{P} x D{D}, B={B}, U={U}, V={V}, b={mbs}, "
                                   f"s={spec.seq_len}", "model": MODELS[args.model][1],
                       "tokens_per_step": tokens_per_step, "parallelism": "cpu (host cores)"},
            "cpu_baseline": {"value": round(value, 3), "unit": "tokens/s", "cores": last["cores"], "kind": "port",
                             "sample": last["sample"], "extrapolated": True},
            "reference_cpu_path": reference_schedule_path(args),
            "c1_measured_step": c1_oracle_step(threads),
            "e2e": {"value": round(value, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1, choices=sorted(SPLITS))
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="zpp", choices=["zpp", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU-baseline leg")
    ap.add_argument("--model", default="gpt-6.2b", choices=sorted(MODELS))
    ap.add_argument("--split", default=None, help="PxD:B:U:V override of the default split for --gpus")
    ap.add_argument("--mb-size", type=int, default=None,
                    help="samples per micro-batch (ParallelConfig.microbatch_samples); default from the split")
    ap.add_argument("--out-dir", default=os.path.join(ROOT, "gpurun_out"))
    ap.add_argument("--rt", default="", help="Runtime keyword overrides for A/B runs, e.g. 'overlap_tail=False'")
    args = ap.parse_args()
    os.makedirs(args.out_dir, exist_ok=True)
    if args.warmup < 3 and args.impl == "zpp":
        print("note: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_zpp(args)


if __name__ == "__main__":
    main()
