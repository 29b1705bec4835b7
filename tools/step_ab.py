"""A/B of Runtime options on the N=1 bench configuration (GPT-6.2B P1 x D1 B8 U2 b2), same process,
alternating A B A B ... so clock / power drift hits both arms equally.

    python tools/step_ab.py 'stream_priority=False' 'stream_priority=True' [--rounds 3 --steps 4]

Each argument is a comma-separated list of Runtime keyword overrides (Python literals)."""
import argparse
import ast
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch  # noqa: E402

from paper_2402_03791_b200.engine import lib  # noqa: E402

if os.environ.get("ZPP_LIB_AB"):  # A/B against another build of the library (tools only)
    lib.LIB_PATH = os.environ["ZPP_LIB_AB"]
from paper_2402_03791_b200 import ModelSpec, ParallelConfig, generate, make_placement  # noqa: E402
from paper_2402_03791_b200.engine import GPTSpec, Runtime  # noqa: E402
from paper_2402_03791_b200.engine.data import synthetic_tokens  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("arms", nargs="+")
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--steps", type=int, default=4)
a = ap.parse_args()
spec = GPTSpec.gpt_6p2b(microbatch_samples=2)
model = ModelSpec(num_layers=spec.num_layers, hidden_size=spec.hidden, seq_len=spec.seq_len)
cfg = ParallelConfig(pp_size=1, dp_size=1, microbatches=8, unit_size=2, microbatch_samples=2)
pl = make_placement(cfg, model)
sched = generate(model, cfg, pl)
tok = synthetic_tokens(1, 1, 8, 2, spec.seq_len, spec.vocab)[0, 0]
ids = tok[:, :, :-1].reshape(8, -1).contiguous().cuda()
lab = tok[:, :, 1:].reshape(8, -1).contiguous().cuda()
arms = [{k: ast.literal_eval(v) for k, v in (kv.split("=") for kv in arm.split(",") if kv)} for arm in a.arms]
res = {i: [] for i in range(len(arms))}
for r in range(a.rounds):
    for i, kw in enumerate(arms):
        rt = Runtime(spec, model, cfg, pl, sched, **kw)
        for _ in range(2):
            rt.step(ids, lab)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(rt.s_comp)
        for _ in range(a.steps):
            rt.step(ids, lab)
        rt.join(rt.s_comp)
        e1.record(rt.s_comp)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        res[i].append(ms)
        print(f"round {r} arm {a.arms[i]!r}: {ms:.1f} ms/step, {32768 / ms * 1e3:.0f} tok/s", flush=True)
        del rt
        torch.cuda.empty_cache()
for i, arm in enumerate(a.arms):
    ms = sorted(res[i])[len(res[i]) // 2]
    print(f"median {arm!r}: {ms:.1f} ms/step  {32768 / ms * 1e3:.0f} tok/s")
