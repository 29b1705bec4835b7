"""Run one GEMM shape a few times (for ncu).  usage: gemm_one.py M N K a_t b_t epi(bf16|f32acc)"""
import sys
import torch
sys.path.insert(0, '.')
import os
from paper_2402_03791_b200.engine import lib
if os.environ.get("ZPP_LIB_AB"):  # A/B against another build of the library (tools only)
    lib.LIB_PATH = os.environ["ZPP_LIB_AB"]
from paper_2402_03791_b200.engine import ops
M, N, K = (int(x) for x in sys.argv[1:4])
at, bt = sys.argv[4] == '1', sys.argv[5] == '1'
ep = sys.argv[6]
ops.preload()
bf = lambda *s: (torch.randn(*s, device='cuda') * 0.05).to(torch.bfloat16)  # noqa: E731
A = bf(K, M) if at else bf(M, K)
B = bf(K, N) if bt else bf(N, K)
C = torch.zeros(M, N, device='cuda', dtype=torch.float32 if ep == 'f32acc' else torch.bfloat16)
e = ops.EPI_F32_ACC if ep == 'f32acc' else ops.EPI_BF16
for _ in range(3):
    ops.gemm(A, B, C, a_t=at, b_t=bt, epilogue=e)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(10):
    ops.gemm(A, B, C, a_t=at, b_t=bt, epilogue=e)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"{M}x{N}x{K} a_t={int(at)} b_t={int(bt)}: {ms*1e3:.1f} us {2*M*N*K/ms/1e9:.1f} TF/s")
