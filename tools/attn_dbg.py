import sys, os, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_03791_b200.engine import ops
b, s, H, D = 1, 128, 2, 64
torch.manual_seed(0)
qkv = torch.randn(b * s, 3 * H * D, device="cuda").to(torch.bfloat16)
out = torch.empty(b * s, H * D, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(b, H, s, device="cuda")
ops.attn_fwd(qkv, out, lse, b, s, H, D)
do = torch.randn(b * s, H * D, device="cuda").to(torch.bfloat16)
dqkv = torch.zeros_like(qkv)
ws = torch.empty(ops.attn_bwd_workspace(b, s, H, D), device="cuda")
ops.attn_bwd(qkv, out, lse, do, dqkv, ws, b, s, H, D)
qf = qkv.float().requires_grad_(True)
q, k, v = qf.view(b, s, 3, H, D).unbind(2)
q, k, v = (t.transpose(1, 2) for t in (q, k, v))
att = (q @ k.transpose(-1, -2)) / math.sqrt(D)
att = att.masked_fill(torch.ones(s, s, device="cuda", dtype=torch.bool).triu(1), float("-inf"))
o = (torch.softmax(att, -1) @ v).transpose(1, 2).reshape(b * s, H * D)
o.backward(do.float())
g = qf.grad.view(b * s, 3, H * D)[:, 0]
d = dqkv.view(b * s, 3, H * D)[:, 0].float()
for r0 in range(0, s, 32):
    print(" ".join(f"{((d[r0:r0+32, c0:c0+32]-g[r0:r0+32, c0:c0+32]).norm()/g[r0:r0+32, c0:c0+32].norm()).item():.2f}" for c0 in range(0, H * D, 32)))
print("ratio", (d.norm() / g.norm()).item())
bad = d[32:64]
for name, cand in [("g32", g[32:64]), ("g0", g[0:32]), ("g64", g[64:96]), ("g96", g[96:128]), ("g32+g0", g[32:64] + g[0:32]), ("2g32", 2 * g[32:64]), ("g32+g64", g[32:64] + g[64:96])]:
    print(name, ((bad - cand).norm() / cand.norm()).item())
diff = bad - g[32:64]
for name, cand in [("g0", g[0:32]), ("g64", g[64:96]), ("g96", g[96:128])]:
    print("diff vs", name, ((diff - cand).norm() / cand.norm()).item(), ((diff + cand).norm() / cand.norm()).item())
