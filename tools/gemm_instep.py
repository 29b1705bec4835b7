"""In-step GEMM efficiency per shape: one GPT-6.2B N=1 bench step (P1 x D1 B8 U2 b2) with every
GEMM bracketed by CUDA events on its stream (ops.PROFILE), aggregated per (M, N, K, layout,
epilogue).  Prints launches, ms per step and TF/s per shape, heaviest first."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_03791_b200.engine import lib  # noqa: E402

if os.environ.get("ZPP_LIB_AB"):  # A/B against another build of the library (tools only)
    lib.LIB_PATH = os.environ["ZPP_LIB_AB"]
from paper_2402_03791_b200 import ModelSpec, ParallelConfig, generate, make_placement  # noqa: E402
from paper_2402_03791_b200.engine import GPTSpec, Runtime, ops  # noqa: E402
from paper_2402_03791_b200.engine.data import synthetic_tokens  # noqa: E402

spec = GPTSpec.gpt_6p2b(microbatch_samples=2)
model = ModelSpec(num_layers=spec.num_layers, hidden_size=spec.hidden, seq_len=spec.seq_len)
cfg = ParallelConfig(pp_size=1, dp_size=1, microbatches=8, unit_size=2, microbatch_samples=2)
pl = make_placement(cfg, model)
rt = Runtime(spec, model, cfg, pl, generate(model, cfg, pl))
tok = synthetic_tokens(1, 1, 8, 2, spec.seq_len, spec.vocab)[0, 0]
ids = tok[:, :, :-1].reshape(8, -1).contiguous().cuda()
lab = tok[:, :, 1:].reshape(8, -1).contiguous().cuda()
if "--no-streamk" in sys.argv:  # A/B: whole tiles only (the last partial wave is not split)
    ops.set_streamk(False)
for _ in range(3):
    rt.step(ids, lab)
torch.cuda.synchronize()
steps = 2
ops.PROFILE.start(time_gemms=True)
for _ in range(steps):
    rt.step(ids, lab)
flops, ms, n, shapes = ops.PROFILE.stop(by_shape=True)
print(f"all GEMMs: {n // steps} launches/step, {ms / steps:.1f} ms/step, {flops / (ms / 1e3) / 1e12:.0f} TF/s")
names = {ops.EPI_BF16: "bf16", ops.EPI_F32_ACC: "f32acc"}
for (M, N, K, at, bt, epi), (cnt, f, t) in sorted(shapes.items(), key=lambda kv: -kv[1][2]):
    print(f"{M:6d} x {N:6d} x {K:6d} a_t={at} b_t={bt} epi={names.get(epi, epi):>6}: {cnt // steps:4d}/step "
          f"{t / steps:7.1f} ms/step {t / cnt * 1e3:7.1f} us  {f / (t / 1e3) / 1e12:6.0f} TF/s")
