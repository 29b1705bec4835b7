"""One causal attention fwd+bwd at GPT-6.2B shape (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_03791_b200.engine import ops
b, s, H, D = 1, 2048, 32, 128
qkv = (torch.randn(b * s, 3 * H * D, device="cuda")).to(torch.bfloat16)
out = torch.empty(b * s, H * D, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(b, H, s, device="cuda")
do = torch.randn(b * s, H * D, device="cuda").to(torch.bfloat16)
dqkv = torch.empty_like(qkv)
ws = torch.empty(ops.attn_bwd_workspace(b, s, H, D), device="cuda")
for _ in range(2):
    ops.attn_fwd(qkv, out, lse, b, s, H, D)
    ops.attn_bwd(qkv, out, lse, do, dqkv, ws, b, s, H, D)
torch.cuda.synchronize()
print("ok")
