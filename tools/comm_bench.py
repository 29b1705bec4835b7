"""Collective bandwidth of the engine's ZeRO / P2P traffic over NVLink (libzpp NCCL C-ABI).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/comm_bench.py

All N ranks form one group (a ZeRO group of size D = N).  Sizes are the per-(stage, unit)
payloads of the bench splits: one GPT-6.2B stage of 8 layers (V=2, P=2: 1.61 G params,
bf16) for AG_PARAM / RS_GRAD, and one [2048, 4096] bf16 activation for the stage-boundary
P2P (rank 0 -> rank 1).  CUDA-event time on the communication stream, median of 5 after 2
warm-ups.  algbw = bytes in the gathered / reduced buffer / t; busbw = algbw * (N-1)/N
(the NCCL convention: bytes each rank moves over its links / t).
"""
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import torch
import torch.distributed as dist

from paper_2402_03791_b200.engine import lib

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
dist.init_process_group("gloo")
lib.load()
lib.load_nccl()
uid = ctypes.create_string_buffer(128)
if rank == 0:
    lib.call("zpp_nccl_unique_id", uid)
obj = [uid.raw]
dist.broadcast_object_list(obj, src=0)
comm = ctypes.c_void_p()
lib.call("zpp_comm_init", obj[0], world, rank, ctypes.byref(comm))
s = torch.cuda.Stream()


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = torch.tensor([statistics.median(ts)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


stage_params = 1_610_612_736 // world * world  # 8 layers x 12 h^2 (h = 4096), divisible by N
per = stage_params // world
full = torch.empty(stage_params, dtype=torch.bfloat16, device="cuda")
send = torch.empty(stage_params, dtype=torch.bfloat16, device="cuda")
recv = torch.empty(per, dtype=torch.bfloat16, device="cuda")
out = {"n_ranks": world, "stage_params": stage_params, "bytes_gathered": stage_params * 2}
ms = timed(lambda: lib.call("zpp_allgather", comm, full[rank * per:(rank + 1) * per].data_ptr(), full.data_ptr(),
                            per, 0, s.cuda_stream))
alg = stage_params * 2 / (ms / 1e3) / 1e9
out["allgather"] = {"ms": round(ms, 3), "algbw_GBs": round(alg, 1), "busbw_GBs": round(alg * (world - 1) / world, 1)}
ms = timed(lambda: lib.call("zpp_reduce_scatter", comm, send.data_ptr(), recv.data_ptr(), per, 0, s.cuda_stream))
alg = stage_params * 2 / (ms / 1e3) / 1e9
out["reduce_scatter"] = {"ms": round(ms, 3), "algbw_GBs": round(alg, 1),
                         "busbw_GBs": round(alg * (world - 1) / world, 1)}
act = torch.empty(2048 * 4096, dtype=torch.bfloat16, device="cuda")


def p2p():
    if rank == 0:
        lib.call("zpp_send", comm, act.data_ptr(), act.numel(), 0, 1, s.cuda_stream)
    elif rank == 1:
        lib.call("zpp_recv", comm, act.data_ptr(), act.numel(), 0, 0, s.cuda_stream)


ms = timed(p2p, reps=10)
out["p2p_activation"] = {"bytes": act.numel() * 2, "ms": round(ms, 4), "GBs": round(act.numel() * 2 / (ms / 1e3) / 1e9, 1)}
if rank == 0:
    print(json.dumps(out), flush=True)
dist.destroy_process_group()
