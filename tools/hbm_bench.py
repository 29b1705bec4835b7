"""HBM-bound kernels at the step's shapes (T = 4096 tokens, h = 4096): achieved GB/s of
algorithmic bytes vs MEASURED_PEAKS.json hbm_gbs.  CUDA events, median of 20 after warm-up."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_03791_b200.engine import lib, ops

if os.environ.get("ZPP_LIB_AB"):  # A/B against another build of the library (tools only)
    lib.LIB_PATH = os.environ["ZPP_LIB_AB"]

T, h = (int(x) for x in sys.argv[1:3]) if len(sys.argv) > 2 else (4096, 4096)
dev = "cuda"
ops.preload()
bf = lambda *s: torch.randn(*s, device=dev).to(torch.bfloat16)  # noqa: E731
x, g, b, dy, dres = bf(T, h), bf(h), bf(h), bf(T, h), bf(T, h)
y, dx = torch.empty_like(x), torch.empty_like(x)
mean, rstd = torch.empty(T, device=dev), torch.empty(T, device=dev)
ws = torch.zeros(ops.layernorm_bwd_workspace(T, 4 * h), device=dev)
dgam, dbet = torch.zeros(h, device=dev), torch.zeros(h, device=dev)
dy4 = bf(T, 4 * h)
db4 = torch.zeros(4 * h, device=dev)
n_opt = 256 * 1024 * 1024
pm, m, v, gr = (torch.zeros(n_opt, device=dev) for _ in range(4))
pb = torch.empty(n_opt, dtype=torch.bfloat16, device=dev)


def t(fn):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts) * 1e3  # us


peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists("MEASURED_PEAKS.json") else 6650.0
rows = [
    ("layernorm_fwd", lambda: ops.layernorm_fwd(x, g, b, y, mean, rstd), 2 * T * h * 2),
    ("layernorm_bwd_dx (+resid)", lambda: ops.layernorm_bwd(dy, x, mean, rstd, g, dx, None, None, None, dresid=dres),
     4 * T * h * 2),
    ("norm_param_grads", lambda: ops.norm_param_grads(dy, x, mean, rstd, dgam, dbet, ws), 2 * T * h * 2),
    ("colsum (bias grad, 4h)", lambda: ops.colsum_acc(dy4, db4, ws), T * 4 * h * 2),
    ("adamw (256 M params)", lambda: ops.adamw(pm, m, v, gr, pb, 1e-4, 0.9, 0.95, 1e-8, 0.1, 1), n_opt * 30),
]
out = {}
for name, fn, byts in rows:
    us = t(fn)
    out[name] = {"us": round(us, 2), "GBs": round(byts / us / 1e3, 1), "frac": round(byts / us / 1e3 / peak, 3)}
    print(f"{name:28s} {us:9.2f} us  {byts / us / 1e3:8.1f} GB/s  {byts / us / 1e3 / peak:5.2f} of {peak:.0f}")
print(json.dumps(out))
