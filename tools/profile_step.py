"""Kernel-time breakdown of one GPT-6.2B-width ZeroPP step (torch.profiler / CUPTI).

    python tools/profile_step.py [--layers L] [--B 8] [--U 2] [--ncu]

With --ncu the step is bracketed by cudaProfilerStart/Stop so that
`ncu --profile-from-start off` captures exactly one step.
"""
import argparse, os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_03791_b200.engine.data import synthetic_tokens as make_tokens
from paper_2402_03791_b200 import ModelSpec, ParallelConfig, generate, make_placement
from paper_2402_03791_b200.engine import GPTSpec, Runtime

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--B", type=int, default=8)
ap.add_argument("--U", type=int, default=2)
ap.add_argument("--mb", type=int, default=2, help="samples per micro-batch (bench default b=2)")
ap.add_argument("--ncu", action="store_true")
ap.add_argument("--gemm-shapes", default=None, help="with --ncu: write M,N,K,algorithmic bytes per GEMM launch")
ap.add_argument("--rt", default="", help="Runtime keyword overrides, e.g. 'aux_stream=False'")
a = ap.parse_args()
import ast
rt_kw = {k: ast.literal_eval(v) for k, v in (kv.split("=") for kv in a.rt.split(",") if kv)}
spec = GPTSpec(num_layers=a.layers, hidden=4096, heads=32, seq_len=2048, microbatch_samples=a.mb)
model = ModelSpec(num_layers=spec.num_layers, hidden_size=spec.hidden, seq_len=spec.seq_len)
cfg = ParallelConfig(pp_size=1, dp_size=1, microbatches=a.B, unit_size=a.U, microbatch_samples=a.mb)
pl = make_placement(cfg, model)
sched = generate(model, cfg, pl)
rt = Runtime(spec, model, cfg, pl, sched, **rt_kw)
t = make_tokens(1, 1, a.B, a.mb, spec.seq_len, spec.vocab)[0, 0]
ids = t[:, :, :-1].reshape(a.B, -1).contiguous().cuda()
lab = t[:, :, 1:].reshape(a.B, -1).contiguous().cuda()
for _ in range(2):
    rt.step(ids, lab)
torch.cuda.synchronize()
if a.ncu:
    from paper_2402_03791_b200.engine import ops
    if a.gemm_shapes:
        ops.PROFILE.shapes = []
    torch.cuda.profiler.start()
    rt.step(ids, lab)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    if a.gemm_shapes:
        with open(a.gemm_shapes, "w") as f:
            for row in ops.PROFILE.shapes:
                f.write(",".join(map(str, row)) + "\n")
    sys.exit(0)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rt.step(ids, lab)
    torch.cuda.synchronize()
tot = collections.Counter(); cnt = collections.Counter()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        name = e.name.split("(")[0].split("<")[0].replace("void ", "").replace("zpp::", "")
        tot[name] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
        cnt[name] += 1
all_us = sum(tot.values())
print(f"{'kernel':40s} {'calls':>6s} {'ms':>9s} {'share':>6s}")
for k, v in tot.most_common():
    print(f"{k[:40]:40s} {cnt[k]:6d} {v/1e3:9.2f} {100*v/all_us:5.1f}%")
print(f"total kernel time {all_us/1e3:.1f} ms")

# inter-kernel idle gaps on the compute stream (CUPTI timestamps)
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
             key=lambda e: e.time_range.start)
gaps = []
for a, b in zip(evs, evs[1:]):
    g = b.time_range.start - a.time_range.end
    if g > 0:
        gaps.append((g, a.name.split("(")[0][:30], b.name.split("(")[0][:30]))
span = evs[-1].time_range.end - evs[0].time_range.start
tot_gap = sum(g for g, _, _ in gaps)
print(f"span {span/1e3:.1f} ms, kernel-to-kernel idle {tot_gap/1e3:.1f} ms over {len(gaps)} gaps "
      f"(median {sorted(g for g,_,_ in gaps)[len(gaps)//2]:.2f} us)")
by = collections.Counter()
for g, a, b in gaps:
    by[(a, b)] += g
for (a, b), g in by.most_common(8):
    print(f"  {g/1e3:7.2f} ms  {a} -> {b}")
