"""GEMM throughput on the GPT-6.2B linear shapes: tcgen05 kernel (1-CTA / CTA-pair) vs cuBLAS."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_03791_b200.engine import ops

T, h = 2048, 4096
shapes = [("qkv fwd", T, 3 * h, h, False, False), ("proj fwd", T, h, h, False, False),
          ("fc1 fwd", T, 4 * h, h, False, False), ("fc2 fwd", T, h, 4 * h, False, False),
          ("fc1 dgrad", T, h, 4 * h, False, True), ("fc2 dgrad", T, 4 * h, h, False, True),
          ("qkv wgrad", 3 * h, h, T, True, True), ("fc1 wgrad", 4 * h, h, T, True, True),
          ("lm_head", T, 50304, h, False, False), ("lm wgrad", 50304, h, T, True, True),
          ("big 8192^3", 8192, 8192, 8192, False, False)]


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


for name, M, N, K, a_t, b_t in shapes:
    a = torch.randn(K, M, device="cuda").to(torch.bfloat16) if a_t else torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(K, N, device="cuda").to(torch.bfloat16) if b_t else torch.randn(N, K, device="cuda").to(torch.bfloat16)
    epi = ops.EPI_F32_ACC if a_t else ops.EPI_BF16
    c = torch.zeros(M, N, device="cuda", dtype=torch.float32 if a_t else torch.bfloat16)
    fl = 2.0 * M * N * K
    res = []
    for cg in (1, 2):
        ops.set_cta_group(cg)
        ms = timeit(lambda: ops.gemm(a, b, c, a_t=a_t, b_t=b_t, epilogue=epi))
        res.append(f"cta{cg} {ms*1e3:7.1f} us {fl/ms/1e9:7.1f} TF/s")
    ops.set_cta_group(0)
    A = a.t() if a_t else a
    B = b if b_t else b.t()
    ms_ref = timeit(lambda: torch.matmul(A, B))
    print(f"{name:10s} {M:6d}x{N:6d}x{K:6d} | " + " | ".join(res) + f" | cuBLAS {fl/ms_ref/1e9:7.1f} TF/s", flush=True)
