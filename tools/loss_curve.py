"""Per-step loss of repeated steps on one fixed synthetic batch (P1 x D1), for a model at full
width with fewer layers: checks the first-step loss is ln(vocab)-ish and how fast it falls.

    python tools/loss_curve.py --model llama-7b --layers 4 --steps 8
"""
import argparse, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch
import bench
from paper_2402_03791_b200 import ModelSpec, ParallelConfig, generate, make_placement
from paper_2402_03791_b200.engine import GPTSpec, Runtime
from paper_2402_03791_b200.engine.data import synthetic_tokens

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama-7b", choices=sorted(bench.MODELS))
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--B", type=int, default=2)
ap.add_argument("--steps", type=int, default=8)
a = ap.parse_args()
spec = getattr(GPTSpec, bench.MODELS[a.model][0])(num_layers=a.layers) if False else None
base = getattr(GPTSpec, bench.MODELS[a.model][0])()
import dataclasses
spec = dataclasses.replace(base, num_layers=a.layers)
model = ModelSpec(num_layers=spec.num_layers, hidden_size=spec.hidden, seq_len=spec.seq_len)
cfg = ParallelConfig(pp_size=1, dp_size=1, microbatches=a.B, unit_size=1)
pl = make_placement(cfg, model)
rt = Runtime(spec, model, cfg, pl, generate(model, cfg, pl))
t = synthetic_tokens(1, 1, a.B, 1, spec.seq_len, spec.vocab)[0, 0]
ids = t[:, :, :-1].reshape(a.B, -1).contiguous().cuda()
lab = t[:, :, 1:].reshape(a.B, -1).contiguous().cuda()
print(f"{a.model} L{a.layers}: ln(vocab) = {math.log(spec.vocab):.4f}")
for k in range(a.steps):
    r = rt.step(ids, lab)
    print(f"step {k + 1}: loss {r.loss_sum.item() / (a.B * spec.tokens_per_microbatch):.5f}", flush=True)
