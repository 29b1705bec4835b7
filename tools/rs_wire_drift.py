"""bf16 vs fp32 wire for RS_GRAD: gradient error against the fp32 oracle at a real width.

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/rs_wire_drift.py [L] [B]

One engine step of a 2-layer GPT-6.2B-width model (h4096, s2048, b=2) at P1 x D4 (B micro-batches
per rank, U=1 so every micro-batch's gradient is reduce-scattered separately: the worst case
for per-hop bf16 rounding), once with each wire; each rank compares its fp32 gradient shard
with the oracle's (evaluated on its own GPU in strict fp32) and prints cosine, max|err|/max|g|
and the 99.9th percentile of |err| / max|g|."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests"))
sys.path.insert(0, os.path.dirname(HERE))
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from engine_harness import flat_stage, oracle_for, params_from_flat, run_engine_step  # noqa: E402
from paper_2402_03791_b200.engine import GPTSpec  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
dist.init_process_group("gloo")
L = int(sys.argv[1]) if len(sys.argv) > 1 else 2
B = int(sys.argv[2]) if len(sys.argv) > 2 else 2
spec = GPTSpec(num_layers=L, hidden=4096, heads=32, seq_len=2048, microbatch_samples=2)
out = {}
for wire in ("bf16", "fp32"):
    rt, (model, cfg, pl, sched), tokens, res = run_engine_step(spec, 1, world, B, 1, 1, rank=rank, world=world,
                                                                timeline=False, rt_kw={"rs_wire": wire})
    out[wire] = {s: rt.captured[s].float().clone() for s in rt.stages}
    lo = rt.z * rt.stages[0].lay.shard_numel
    ns = rt.stages[0].lay.shard_numel
    del rt, res
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
# oracle params: the deterministic init, gathered from the numpy restatement (small: 2 layers)
from engine_harness import oracle_params  # noqa: E402
params = oracle_params(spec, cfg, pl)
_, grads_o, _ = oracle_for(spec, cfg, pl, tokens[0], params=params, device="cuda")
g_ref = flat_stage(spec, cfg, pl, 0, grads_o)[lo:lo + ns]
gmax = g_ref.abs().max().item()
for wire, gs in out.items():
    g = gs[0].to(g_ref.device)
    err = (g - g_ref).abs()
    cos = torch.nn.functional.cosine_similarity(g, g_ref, dim=0).item()
    q = torch.quantile(err[torch.randperm(err.numel(), device=err.device)[:1 << 22]] / gmax, 0.999).item()
    print(f"rank {rank} wire {wire}: cos {cos:.7f}  max|err|/max|g| {err.max().item() / gmax:.3e}  "
          f"p99.9 {q:.3e}", flush=True)
d = (out["bf16"][0] - out["fp32"][0]).abs().max().item()
print(f"rank {rank}: max|g_bf16wire - g_fp32wire| / max|g| = {d / gmax:.3e}", flush=True)
dist.barrier()
dist.destroy_process_group()
