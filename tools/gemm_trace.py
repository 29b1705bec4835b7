"""Timeline of one GEMM launch (debug build: make -C paper_2402_03791_b200/csrc trace).  usage: gemm_trace.py M N K a_t b_t [bf16|f32|f32acc]"""
import ctypes
import os
import sys

import numpy as np
import torch


sys.path.insert(0, '.')
from paper_2402_03791_b200.engine import lib  # noqa: E402

lib.LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libzpp_trace.so")
from paper_2402_03791_b200.engine import ops  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
at, bt = sys.argv[4] == '1', sys.argv[5] == '1'
ops.preload()
bf = lambda *s: (torch.randn(*s, device='cuda') * 0.05).to(torch.bfloat16)  # noqa: E731
A = bf(K, M) if at else bf(M, K)
B = bf(K, N) if bt else bf(N, K)
epi = sys.argv[6] if len(sys.argv) > 6 else "bf16"
C = torch.zeros(M, N, device='cuda', dtype=torch.bfloat16 if epi == "bf16" else torch.float32)
EPI = {"bf16": ops.EPI_BF16, "f32": ops.EPI_F32, "f32acc": ops.EPI_F32_ACC}[epi]
L = lib.load()
L.zpp_gemm_trace_dump.restype = ctypes.c_longlong
buf = np.zeros(148 * 32 * 6, dtype=np.uint64)
for _ in range(3):
    ops.gemm(A, B, C, a_t=at, b_t=bt, epilogue=EPI)
    torch.cuda.synchronize()
    L.zpp_gemm_trace_dump(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_longlong(buf.size))
t = buf.reshape(148, 32, 6).astype(np.int64)
flag = (t[:, :, 5] >> 63) & 1
t[:, :, 5] &= (1 << 62) - 1
valid = t[:, :, 1] > 0
t0 = t[:, :, 1][valid].min()
print("cta it item  mma0  mma1 | epi0 epiacc epi1 (us from launch)")
for c in list(range(0, 148, 2))[:int(os.environ.get("ROWS", "12"))]:
    line = []
    for i in range(32):
        if t[c, i, 1] == 0:
            break
        r = t[c, i]
        line.append(f"[{r[0]}: m {(r[1]-t0)/1e3:.1f}-{(r[2]-t0)/1e3:.1f} e {(r[3]-t0)/1e3:.1f}/{(r[4]-t0)/1e3:.1f}-{(r[5]-t0)/1e3:.1f}{'p' if flag[c,i] else ''}]")
    print(c, " ".join(line))
end = (t[:, :, 5][t[:, :, 5] > 0] - t0).max() / 1e3
print("last epilogue end (us):", end)
