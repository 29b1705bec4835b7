"""wgrad GEMM shapes under each epilogue: is the fp32 reduce-add the limiter?"""
import sys
import torch
sys.path.insert(0, '.')
from paper_2402_03791_b200.engine import ops
ops.preload()
bf = lambda *s: (torch.randn(*s, device='cuda') * 0.05).to(torch.bfloat16)  # noqa: E731
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device='cuda')
K_TOK = int(sys.argv[1]) if len(sys.argv) > 1 else 4096  # tokens per micro-batch (b = 2: 4096)
for name, M, N, K in [("qkv", 12288, 4096, K_TOK), ("proj", 4096, 4096, K_TOK), ("fc1", 16384, 4096, K_TOK),
                      ("fc2", 4096, 16384, K_TOK)]:
    A, B = bf(K, M), bf(K, N)
    out = []
    for ep, dt in ((ops.EPI_F32_ACC, torch.float32), (ops.EPI_F32, torch.float32), (ops.EPI_BF16, torch.bfloat16)):
        C = torch.zeros(M, N, device='cuda', dtype=dt)
        for _ in range(3):
            ops.gemm(A, B, C, a_t=True, b_t=True, epilogue=ep)
        ts = []
        for _ in range(10):
            flush.zero_()
            s, t = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record(); ops.gemm(A, B, C, a_t=True, b_t=True, epilogue=ep); t.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(t))
        ts.sort()
        out.append(ts[5] * 1e3)
    f = 2 * M * N * K / 1e6
    print(f"{name:5s} {M}x{N}x{K}: f32acc {out[0]:6.1f} us ({f/out[0]:6.0f} TF/s)  f32 {out[1]:6.1f} us ({f/out[1]:6.0f})"
          f"  bf16 {out[2]:6.1f} us ({f/out[2]:6.0f})", flush=True)
