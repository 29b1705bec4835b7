"""Run one GEMM shape repeatedly (for ncu): python tools/gemm_one.py M N K a_t b_t cg [iters]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_03791_b200.engine import ops
M, N, K, a_t, b_t, cg = (int(x) for x in sys.argv[1:7])
iters = int(sys.argv[7]) if len(sys.argv) > 7 else 3
a = torch.randn(K, M, device="cuda").to(torch.bfloat16) if a_t else torch.randn(M, K, device="cuda").to(torch.bfloat16)
b = torch.randn(K, N, device="cuda").to(torch.bfloat16) if b_t else torch.randn(N, K, device="cuda").to(torch.bfloat16)
epi = ops.EPI_F32_ACC if a_t else ops.EPI_BF16
c = torch.zeros(M, N, device="cuda", dtype=torch.float32 if a_t else torch.bfloat16)
ops.set_cta_group(cg)
for _ in range(iters):
    ops.gemm(a, b, c, a_t=bool(a_t), b_t=bool(b_t), epilogue=epi)
torch.cuda.synchronize()
print("ok")
