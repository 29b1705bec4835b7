"""Where does a multi-rank step wait?  Runs the bench configuration for --gpus N (torchrun)
for a few steps and prints, per rank, the compute-stream waits of the last step (kind,
task, ms), largest first.

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/waits.py --gpus 4
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch
import torch.distributed as dist

import bench
from paper_2402_03791_b200 import ModelSpec, ParallelConfig, generate, make_placement
from paper_2402_03791_b200.engine import GPTSpec, Runtime
from paper_2402_03791_b200.engine.data import synthetic_tokens

ap = argparse.ArgumentParser()
ap.add_argument("--gpus", type=int, default=1)
ap.add_argument("--split", default=None)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--top", type=int, default=12)
args = ap.parse_args()
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
if world > 1:
    dist.init_process_group("gloo")
args.mb_size = None
P, D, B, U, V, mb = bench._split(args)
spec = GPTSpec.gpt_6p2b(microbatch_samples=mb)
model = ModelSpec(num_layers=spec.num_layers, hidden_size=spec.hidden, seq_len=spec.seq_len)
cfg = ParallelConfig(pp_size=P, dp_size=D, microbatches=B, unit_size=U, stages_per_device=V,
                     microbatch_samples=mb)
pl = make_placement(cfg, model)
sched = generate(model, cfg, pl)
rt = Runtime(spec, model, cfg, pl, sched, rank=rank, world=world, timeline=True)
toks = synthetic_tokens(1, D, B, mb, spec.seq_len, spec.vocab)[0]
ids = toks[rt.z, :, :, :-1].reshape(B, -1).contiguous().cuda()
lab = toks[rt.z, :, :, 1:].reshape(B, -1).contiguous().cuda()
for _ in range(args.steps):
    res = rt.step(ids, lab)
res = rt.finish_timing(res)
if world > 1:
    dist.barrier()
for r in range(world):
    if r == rank:
        w = sorted(res.waits, key=lambda x: -x[2])
        tot = {k: sum(ms for kk, _, ms in res.waits if kk == k) for k in ("zero", "p2p")}
        print(f"rank {rank} (p={rt.p} z={rt.z}) step {res.step_ms:.1f} ms  zero {tot['zero']:.2f} ms  "
              f"p2p {tot['p2p']:.2f} ms", flush=True)
        for k, tid, ms in w[:args.top]:
            print(f"   {k:4s} {ms:8.3f} ms  {tid}", flush=True)
    if world > 1:
        dist.barrier()
if world > 1:
    dist.destroy_process_group()
