"""Causal attention timing at GPT-6.2B shape (b1 s2048 H32 d128): tcgen05 vs mma.sync kernels."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_03791_b200.engine import ops
b, s, H, D = 1, 2048, 32, 128
if len(sys.argv) > 1:
    b, s, H, D = (int(x) for x in sys.argv[1:5])
qkv = (torch.randn(b * s, 3 * H * D, device="cuda")).to(torch.bfloat16)
out = torch.empty(b * s, H * D, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(b, H, s, device="cuda")
do = torch.randn(b * s, H * D, device="cuda").to(torch.bfloat16)
dqkv = torch.empty_like(qkv)
ws = torch.empty(ops.attn_bwd_workspace(b, s, H, D), device="cuda")
flops_fwd = 4.0 * b * H * s * s * D / 2  # causal
def timeit(fn, iters=20):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters
for impl, name in ((0, "tc-2tile"), (2, "tc-1tile"), (1, "mma.sync")):
    ops.set_attn_impl(impl)
    f = timeit(lambda: ops.attn_fwd(qkv, out, lse, b, s, H, D))
    bw = timeit(lambda: ops.attn_bwd(qkv, out, lse, do, dqkv, ws, b, s, H, D))
    print(f"{name:9s} fwd {f*1e3:8.1f} us {flops_fwd/f/1e9:7.1f} TF/s | bwd {bw*1e3:8.1f} us {2.5*flops_fwd/bw/1e9:7.1f} TF/s", flush=True)
ops.set_attn_impl(0)
