"""Sustained GEMM under the power cap: CTA pairs (cta_group::2, 32 KB of operand traffic per SM
per k-block) vs single-CTA tiles (48 KB): same FLOPs, 1.5x the L2->SM bytes.  Samples SM clock
and board power with nvidia-smi while each arm runs back to back for ~6 s.

    python tools/gemm_power.py [M N K]"""
import os
import statistics
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_03791_b200.engine import ops  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (4096, 16384, 4096)
ops.preload()
A = (torch.randn(M, K, device="cuda") * 0.05).to(torch.bfloat16)
B = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for cg in (2, 1, 2, 1):
    ops.set_cta_group(cg)
    for _ in range(20):
        ops.gemm(A, B, C)
    torch.cuda.synchronize()
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-lms", "100"], stdout=subprocess.PIPE, text=True)
    n, t0 = 0, time.time()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < 6:
        for _ in range(50):
            ops.gemm(A, B, C)
        n += 50
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    smi.terminate()
    rows = [l.split(",") for l in smi.communicate()[0].splitlines() if l.strip()]
    clk = statistics.median(float(r[0]) for r in rows[5:])
    pw = statistics.median(float(r[1]) for r in rows[5:])
    tf = 2.0 * M * N * K * n / (e0.elapsed_time(e1) / 1e3) / 1e12
    print(f"cta_group {cg}: {tf:7.1f} TF/s  sm {clk:.0f} MHz  {pw:.0f} W  ({tf / clk * 1e3:.3f} TF/s per GHz)", flush=True)
ops.set_cta_group(0)
