"""End-to-end ZeroPP step on one B200 vs the CPU fp32 oracle (tolerances in engine_harness)."""

import os
import shutil
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

from engine_harness import (LOSS_RTOL, check_init_sample, compare_shards, oracle_for,  # noqa: E402
                            params_from_flat, rank_tokens, run_engine_step)
from paper_2402_03791_b200.engine import GPTSpec, execute  # noqa: E402

# Reduced-depth models at the BENCH widths: the exact kernel
# shapes the headline runs (head_dim 128, s = 2048 / 4096, b = 2, vocab 50304 / 32000).
WIDE = {
    "gpt-6.2b": lambda **kw: GPTSpec(num_layers=2, hidden=4096, heads=32, seq_len=2048, microbatch_samples=2, **kw),
    "llama-7b": lambda **kw: GPTSpec(num_layers=2, hidden=4096, heads=32, seq_len=4096, vocab=32000, arch="llama",
                                     ffn_hidden=11008, **kw),
    "gpt-13b": lambda **kw: GPTSpec(num_layers=2, hidden=5120, heads=40, seq_len=2048, **kw),  # gpt_13b, 2 layers
}


@pytest.mark.parametrize("B,U,V", [(8, 4, 2), (4, 2, 1), (8, 8, 4)])
def test_single_gpu_step_matches_oracle(B, U, V):
    spec = GPTSpec.tiny()
    rt, (model, cfg, pl, sched), tokens, res = run_engine_step(spec, 1, 1, B, U, V)
    loss = res[0].loss_sum.item() / (B * spec.tokens_per_microbatch)
    loss_o, grads_o, new_o = oracle_for(spec, cfg, pl, tokens[0])
    assert abs(loss - loss_o) / loss_o <= LOSS_RTOL, (loss, loss_o)
    fails = compare_shards(spec, cfg, pl, rt, grads_o, new_o)
    assert not fails, fails
    # every compute task ran on the device, in schedule order, with measured times
    r = res[0]
    assert set(r.task_times) == set(sched.per_device[0])
    starts = [r.task_times[t][0] for t in sched.per_device[0] if t.is_compute]
    assert starts == sorted(starts)


@pytest.mark.parametrize("B,U,V", [(8, 4, 2), (4, 4, 4)])
def test_recompute_step_matches_oracle(B, U, V):
    """R tasks (recompute=full) re-run early-round stage forwards before B (schedules.py:454-474)."""
    from paper_2402_03791_b200 import RecomputeMode, TaskKind
    spec = GPTSpec.tiny()
    rt, (model, cfg, pl, sched), tokens, res = run_engine_step(spec, 1, 1, B, U, V,
                                                                recompute=RecomputeMode.FULL)
    assert any(t.kind is TaskKind.R for t in sched.per_device[0])
    loss = res[0].loss_sum.item() / (B * spec.tokens_per_microbatch)
    loss_o, grads_o, new_o = oracle_for(spec, cfg, pl, tokens[0])
    assert abs(loss - loss_o) / loss_o <= LOSS_RTOL, (loss, loss_o)
    assert not compare_shards(spec, cfg, pl, rt, grads_o, new_o)


@pytest.mark.parametrize("B,U,V,recompute", [(4, 2, 2, False), (8, 4, 2, True), (4, 4, 1, False)])
def test_llama_step_matches_oracle(B, U, V, recompute):
    """LLaMA block (RMSNorm, SwiGLU, RoPE, no biases) through the same ZeroPP step."""
    from paper_2402_03791_b200 import RecomputeMode
    spec = GPTSpec.tiny_llama()
    kw = {"recompute": RecomputeMode.FULL} if recompute else {}
    rt, (model, cfg, pl, sched), tokens, res = run_engine_step(spec, 1, 1, B, U, V, **kw)
    loss = res[0].loss_sum.item() / (B * spec.tokens_per_microbatch)
    loss_o, grads_o, new_o = oracle_for(spec, cfg, pl, tokens[0])
    assert abs(loss - loss_o) / loss_o <= LOSS_RTOL, (loss, loss_o)
    fails = compare_shards(spec, cfg, pl, rt, grads_o, new_o)
    assert not fails, fails


def test_measured_timeline_is_a_sim_result():
    """execute() with a timeline runtime returns the SimResult superset."""
    from paper_2402_03791_b200 import render_timeline
    from paper_2402_03791_b200.engine.timeline import calibrate, predict
    spec = GPTSpec.tiny()
    rt, (model, cfg, pl, sched), tokens, res = run_engine_step(spec, 1, 1, 8, 4, 2, steps=2)
    r = res[1]
    assert set(r.task_times) == set(sched.tasks())
    assert 0 < r.per_device_busy[0] <= r.makespan <= r.step_ms * 1.001
    assert r.per_device_idle[0] == r.makespan - r.per_device_busy[0]
    assert r.bubble_ratios[0] >= 0 and r.tokens_per_s > 0 and 0 < r.mfu < 1
    assert r.peak_mem_measured[0] > 0 and r.peak_mem[0] > 0
    assert abs(r.loss - r.loss_sum.item() / (8 * spec.tokens_per_microbatch)) < 1e-6
    txt = render_timeline(r.sim, sched)
    assert txt.startswith("makespan=") and "d0" in txt
    fitted, costs = calibrate(r.sim, sched, model, pl)
    pred = predict(sched, fitted, costs, cfg, pl)
    assert pred.makespan > 0


def test_loss_decreases_over_steps():
    spec = GPTSpec.tiny(lr=1e-3)
    B = 4
    rt, _, tokens, res = run_engine_step(spec, 1, 1, B, 2, 1, steps=1, timeline=False)
    # repeat the same batch: the loss must go down under AdamW
    from engine_harness import rank_tokens
    from paper_2402_03791_b200.engine import execute
    ids, labels = (x.cuda() for x in rank_tokens(tokens[0], 0))
    losses = []
    for _ in range(6):
        r = execute(rt.sched, rt.model, rt.cfg, rt.pl, rt, ids, labels)
        losses.append(r.loss_sum.item() / (B * spec.tokens_per_microbatch))
    assert losses[-1] < losses[0] - 0.1, losses


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs 4 GPUs (run via gpurun --gpus 4)")
@pytest.mark.parametrize("P,D,B,U,V,wire", [(2, 2, 8, 4, 2, "bf16"), (4, 1, 8, 4, 1, "bf16"), (1, 4, 4, 2, 2, "bf16"),
                                            (2, 2, 8, 4, 2, "fp32"), (1, 4, 4, 2, 2, "fp32")])
def test_multi_gpu_step_matches_oracle(tmp_path, P, D, B, U, V, wire):
    here = os.path.dirname(os.path.abspath(__file__))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P * D}",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(here, "dist_worker.py"),
           str(P), str(D), str(B), str(U), str(V), str(tmp_path), "1", "dp_outer", wire]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    for rank in range(P * D):
        txt = (tmp_path / f"rank{rank}.txt").read_text()
        assert txt.startswith("OK"), txt


@pytest.mark.parametrize("n,P,D,B,U,V,mode", [
    (2, 1, 1, 4, 2, 2, "dp_outer"), (2, 1, 1, 4, 2, 2, "zero1_outer"),
    (2, 2, 1, 8, 4, 2, "dp_outer"), (2, 1, 2, 4, 2, 1, "zero1_outer"), (2, 2, 1, 8, 4, 1, "zero1_outer")])
def test_outer_dp_step_matches_oracle(tmp_path, n, P, D, B, U, V, mode):
    """n emulated nodes x (P x D): AR_GRAD (DP outer) or RS_GRAD_INTER + AG_PARAM_INTER
    (ZeRO-1 outer) over the replicas (schedules.py:80-87, 144-163, 425-429)."""
    world = n * P * D
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (run via gpurun --gpus {world})")
    here = os.path.dirname(os.path.abspath(__file__))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29534", os.path.join(here, "dist_worker.py"),
           str(P), str(D), str(B), str(U), str(V), str(tmp_path), str(n), mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    for rank in range(world):
        f = tmp_path / f"rank{rank}.txt"
        txt = f.read_text() if f.exists() else "no result"
        assert txt.startswith("OK"), txt + r.stdout[-2000:] + r.stderr[-2000:]
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("P,D,B,U,V,arm", [(1, 1, 4, 2, 1, "noearly"), (1, 1, 4, 2, 2, "noearly"),
                                           (2, 2, 8, 4, 2, "noearly"), (1, 4, 4, 2, 2, "noearly"),
                                           (2, 1, 8, 4, 2, "noearly"), (1, 2, 4, 2, 2, "notail"),
                                           (2, 2, 8, 4, 2, "notail")])
def test_early_optimizer_is_bit_identical(tmp_path, P, D, B, U, V, arm):
    """3 steps with the early (chunked, overlapped) optimizer == 3 steps without it, bit for
    bit: losses, fp32 masters and bf16 shards on every rank.  At D > 1 the early arm also runs
    each step's tail (last RS_GRAD + AdamW) into the next step (Runtime(overlap_tail=True)); the
    ``notail`` cases compare that against the same early optimizer with a serial tail."""
    world = P * D
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (run via gpurun --gpus {world})")
    here = os.path.dirname(os.path.abspath(__file__))
    worker = os.path.join(here, "dist_worker_ab.py")
    args = [str(x) for x in (P, D, B, U, V, 3)] + [str(tmp_path), arm]
    if world == 1:
        cmd = [sys.executable, worker] + args
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr=127.0.0.1", "--master-port=29535", worker] + args
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    for rank in range(world):
        f = tmp_path / f"rank{rank}.txt"
        txt = f.read_text() if f.exists() else "no result"
        assert txt.startswith("OK"), txt + r.stdout[-2000:] + r.stderr[-2000:]
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


def test_cuda_graph_step_is_bit_identical():
    """Runtime(cuda_graph=True): steps 2.. replay a captured graph of the task list up to OPT; 4 steps
    give the same fp32 masters / bf16 params bit for bit as 4 eager steps."""
    spec = GPTSpec.tiny()
    out = {}
    for mode in ("0", "1"):
        rt, _, _, res = run_engine_step(spec, 1, 1, 4, 2, 2, steps=4, timeline=False,
                                        rt_kw={"cuda_graph": mode == "1", "early_opt": False})
        assert rt.graph_mode == (mode == "1") and (rt._graph is not None) == (mode == "1")
        out[mode] = ([r.loss_sum.item() for r in res],
                     {s: (st.master.cpu(), st.shard_bf16.cpu()) for s, st in rt.stages.items()})
        del rt
        torch.cuda.synchronize()
    for s in out["0"][1]:
        assert torch.equal(out["0"][1][s][0], out["1"][1][s][0]), f"stage {s} master"
        assert torch.equal(out["0"][1][s][1], out["1"][1][s][1]), f"stage {s} bf16"
    for a, b in zip(out["0"][0], out["1"][0]):
        assert abs(a - b) <= 1e-6 * abs(a)


def test_oracle_device_independent():
    """The fp32 oracle gives the same step on CPU and on cuda:0 (TF32 off), so the production-width
    tests below may evaluate it on the GPU."""
    spec = GPTSpec.tiny()
    from engine_harness import build
    from oracle.gpt_oracle import make_tokens
    model, cfg, pl, sched = build(spec, 1, 1, 4, 2, 2)
    tokens = make_tokens(1, 1, 4, 1, spec.seq_len, spec.vocab)
    l_c, g_c, n_c = oracle_for(spec, cfg, pl, tokens[0])
    l_g, g_g, n_g = oracle_for(spec, cfg, pl, tokens[0], device="cuda")
    assert abs(l_c - l_g) <= 1e-5 * l_c
    for k in g_c:
        ref = g_c[k]
        assert (g_g[k].cpu() - ref).abs().max().item() <= 1e-4 * ref.abs().max().item() + 1e-9, k
        # AdamW step 1 moves every element by ~lr*sign(g): near-zero grads may flip sign
        d = (n_g[k].cpu() - n_c[k]).abs()
        assert d.max().item() <= 2 * spec.lr and (d > 1e-6).float().mean().item() < 1e-3, k


@pytest.mark.parametrize("name,B,U,V", [("gpt-6.2b", 2, 1, 2), ("llama-7b", 2, 1, 1), ("gpt-13b", 2, 2, 1)])
def test_production_width_step_matches_oracle(name, B, U, V):
    """One ZeroPP step of a 2-layer model at the bench's own widths vs the fp32 oracle, with the
    same tolerances as the tiny tests (engine_harness), per stage and per tensor."""
    spec = WIDE[name]()
    rt, (model, cfg, pl, sched), tokens, res = run_engine_step(spec, 1, 1, B, U, V, snapshot_init=True,
                                                                timeline=False)
    params = params_from_flat(spec, cfg, pl, rt.init_master)
    assert not check_init_sample(spec, cfg, pl, params)
    loss = res[0].loss_sum.item() / (B * spec.tokens_per_microbatch)
    loss_o, grads_o, new_o = oracle_for(spec, cfg, pl, tokens[0], params=params, device="cuda")
    del params
    report = []
    fails = compare_shards(spec, cfg, pl, rt, grads_o, new_o, report=report)
    worst = min(report, key=lambda r: r[3])
    print(f"{name}: loss {loss:.5f} oracle {loss_o:.5f}; {len(report)} tensors, worst cos {worst}")
    for row in sorted(report, key=lambda r: -r[4] / r[5])[:5]:
        print(f"   {row[1]}[{row[2]}] cos {row[3]:.6f} maxdiff {row[4]:.3e} = {row[4] / row[5]:.4f} of max|g| {row[5]:.3e}")
    assert abs(loss - loss_o) / loss_o <= LOSS_RTOL, (loss, loss_o)
    assert not fails, fails


@pytest.mark.parametrize("name", ["gpt-6.2b", "llama-7b"])
def test_no_causal_leak_heldout_batch(name):
    """Five steps on batch A, then the loss on a fresh random batch B must stay >= 0.95 ln V:
    random tokens carry no learnable structure, so only a causal-mask leak (position t seeing
    token t+1) could lower it.  Batch A's own loss must fall (the model does learn)."""
    import math
    from oracle.gpt_oracle import make_tokens
    spec = WIDE[name](lr=3e-4)
    B = 2
    rt, _, tokens, res = run_engine_step(spec, 1, 1, B, 1, 1, timeline=False)
    denom = B * spec.tokens_per_microbatch
    ids, labels = (x.cuda() for x in rank_tokens(tokens[0], 0))
    train = [res[0].loss_sum.item() / denom]
    for _ in range(5):
        train.append(execute(rt.sched, rt.model, rt.cfg, rt.pl, rt, ids, labels).loss_sum.item() / denom)
    fresh = make_tokens(1, 1, B, spec.microbatch_samples, spec.seq_len, spec.vocab, seed=12345)
    fid, flab = (x.cuda() for x in rank_tokens(fresh[0], 0))
    held = execute(rt.sched, rt.model, rt.cfg, rt.pl, rt, fid, flab).loss_sum.item() / denom
    print(f"{name}: train {[round(x, 4) for x in train]} held-out {held:.4f} lnV {math.log(spec.vocab):.4f}")
    assert train[-1] < train[0] - 0.1, train
    assert held >= 0.95 * math.log(spec.vocab), (held, train)
