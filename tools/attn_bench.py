"""Causal attention timing (default: GPT-6.2B in-step shape b2 s2048 H32 d128).

usage: python tools/attn_bench.py [b s H D]   -- CUDA-event time per call, useful TF/s
(causal FLOPs: fwd 4*b*H*s^2*d/2, bwd 2.5x fwd)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_03791_b200.engine import lib, ops  # noqa: E402

if os.environ.get("ZPP_LIB_AB"):  # A/B against another build of the library (tools only)
    lib.LIB_PATH = os.environ["ZPP_LIB_AB"]

b, s, H, D = 2, 2048, 32, 128
if len(sys.argv) > 1:
    b, s, H, D = (int(x) for x in sys.argv[1:5])
ops.preload()
qkv = (torch.randn(b * s, 3 * H * D, device="cuda")).to(torch.bfloat16)
out = torch.empty(b * s, H * D, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(b, H, s, device="cuda")
do = torch.randn(b * s, H * D, device="cuda").to(torch.bfloat16)
dqkv = torch.empty_like(qkv)
ws = torch.empty(ops.attn_bwd_workspace(b, s, H, D), device="cuda")
flops_fwd = 4.0 * b * H * s * s * D / 2


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


f = timeit(lambda: ops.attn_fwd(qkv, out, lse, b, s, H, D))
bw = timeit(lambda: ops.attn_bwd(qkv, out, lse, do, dqkv, ws, b, s, H, D))
print(f"b{b} s{s} H{H} d{D}: fwd {f*1e3:8.1f} us {flops_fwd/f/1e9:7.1f} TF/s | "
      f"bwd {bw*1e3:8.1f} us {2.5*flops_fwd/bw/1e9:7.1f} TF/s", flush=True)
