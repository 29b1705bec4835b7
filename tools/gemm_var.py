import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_03791_b200.engine import ops
def timeit(fn, iters=20):
    for _ in range(3): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters
M, N, K = 2048, 12288, 4096
a = torch.randn(M, K, device="cuda").to(torch.bfloat16); b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
c = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
ref = (a.float() @ b.float().t())
for cg in (1, 2):
    for var in (0, 1, 2):
        ops.set_cta_group(cg)
        ms = timeit(lambda: ops.gemm(a, b, c, epilogue=ops.EPI_BF16 | (var << 8)))
        err = ((c.float() - ref).norm() / ref.norm()).item()
        print(f"cg{cg} var{var}: {2*M*N*K/ms/1e9:7.1f} TF/s  relerr {err:.2e}", flush=True)
