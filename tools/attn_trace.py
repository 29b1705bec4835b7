"""Phase timeline of attention-backward CTA 0 from the ZPP_TRACE debug build
(make -C paper_2402_03791_b200/csrc trace -> tools/libzpp_trace.so).  clock64 cycles.

usage: python tools/attn_trace.py [b s H D]"""
import ctypes
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from paper_2402_03791_b200.engine import lib  # noqa: E402

lib.LIB_PATH = os.path.join(HERE, os.environ.get("ZPP_TRACE_LIB", "libzpp_trace.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_03791_b200.engine import ops  # noqa: E402

b, s, H, D = 2, 2048, 32, 128
if len(sys.argv) > 1:
    b, s, H, D = (int(x) for x in sys.argv[1:5])
ops.preload()
qkv = torch.randn(b * s, 3 * H * D, device="cuda").to(torch.bfloat16)
out = torch.empty(b * s, H * D, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(b, H, s, device="cuda")
do = torch.randn(b * s, H * D, device="cuda").to(torch.bfloat16)
dqkv = torch.empty_like(qkv)
ws = torch.empty(ops.attn_bwd_workspace(b, s, H, D), device="cuda")
ops.attn_fwd(qkv, out, lse, b, s, H, D)
for _ in range(3):
    ops.attn_bwd(qkv, out, lse, do, dqkv, ws, b, s, H, D)
torch.cuda.synchronize()
buf = np.zeros((2, 8, 64), dtype=np.uint64)
so = lib.load()
so.zpp_debug_attn_trace.argtypes = [ctypes.c_void_p]
lib.check(so.zpp_debug_attn_trace(buf.ctypes.data), "trace")
names = {0: ["mma:wait_ds", "mma:ds_ok", "mma:S_issued", "mma:dP_issued",
             "sm:wait_S", "sm:S_ok", "sm:wait_dP", "sm:arrived"],
         1: ["mma:wait_ds", "mma:ds_ok", "mma:dV_dK_issued", "mma:SP_issued",
             "sm:wait_SP", "sm:SP_ok", "sm:wait_dsfree", "sm:arrived"]}
for k, kname in ((0, "dq"), (1, "dkdv")):
    t = buf[k].astype(np.int64)
    if not t.any():
        continue
    t0 = t[t > 0].min()  # includes the entry stamp
    n = int((t[7, :63] > 0).sum())
    ev = t[:, 63]
    print(f"== {kname} CTA 0 events: entry {ev[0]-t0} setup {ev[1]-t0} inputs {ev[2]-t0} loop_done {ev[4]-t0} "
          f"epilogue_done {ev[5]-t0}")
    print(f"== {kname} kernel, CTA 0, {n} tiles (cycles from first stamp)")
    print("tile " + " ".join(f"{x:>13s}" for x in names[k]))
    for j in range(n):
        print(f"{j:4d} " + " ".join(f"{(t[i, j] - t0) if t[i, j] else 0:13d}" for i in range(8)))
    per = np.diff(t[7, :n])
    print(f"median softmax-arrive period {np.median(per):.0f} cycles")
