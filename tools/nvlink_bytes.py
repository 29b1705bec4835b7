"""NVLink bytes of a ZeroPP step, from the GPUs' own hardware counters (NVML field values
NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES / _RCV_BYTES per link, or the older THROUGHPUT_DATA_TX / _RX), against
the bytes the executor hands to NCCL (AG_PARAM / RS_GRAD, ``StepResult.nccl_bytes_intra``) and
the stage-boundary P2P bytes it sends.  No profiler and no kernel replay: the counters are read
before and after K steps on every rank.

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/nvlink_bytes.py --gpus 4
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_2402_03791_b200 import ModelSpec, ParallelConfig, TaskKind, generate, make_placement  # noqa: E402
from paper_2402_03791_b200.engine import GPTSpec, Runtime  # noqa: E402
from paper_2402_03791_b200.engine.data import synthetic_tokens  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--gpus", type=int, default=2)
ap.add_argument("--split", default=None)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--model", default="gpt-6.2b")
ap.add_argument("--mb-size", type=int, default=None)
args = ap.parse_args()
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("gloo")

pynvml.nvmlInit()
uuid = str(torch.cuda.get_device_properties(local).uuid)
handle = None
for i in range(pynvml.nvmlDeviceGetCount()):
    h = pynvml.nvmlDeviceGetHandleByIndex(i)
    u = pynvml.nvmlDeviceGetUUID(h)
    u = u.decode() if isinstance(u, bytes) else u
    if u.replace("GPU-", "") == uuid.replace("GPU-", ""):
        handle = h
assert handle is not None, f"no NVML device with uuid {uuid}"
LINKS = 18  # NVLink 5 links per B200


def counters():
    """{name: bytes} summed over links: the per-link NVLink byte counters
    (NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES / _RCV_BYTES, scope = link), else the older throughput
    counters (KiB); None where the driver does not expose a field."""
    out = {}
    for name, fid in (("xmit", pynvml.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES),
                      ("rcv", pynvml.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES)):
        vals = pynvml.nvmlDeviceGetFieldValues(handle, [(fid, link) for link in range(LINKS)])
        ok = [int(v.value.ullVal) for v in vals if v.nvmlReturn == 0]
        out[name] = sum(ok) if ok else None
        out[name + "_links"] = len(ok)
    for name, fid in (("data_tx", pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX),
                      ("data_rx", pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX)):
        v = pynvml.nvmlDeviceGetFieldValues(handle, [fid])[0]
        out[name] = int(v.value.ullVal) * 1024 if v.nvmlReturn == 0 else None
    return out


P, D, B, U, V, mbs = bench._split(args)
spec = getattr(GPTSpec, bench.MODELS[args.model][0])(microbatch_samples=mbs)
model = ModelSpec(num_layers=spec.num_layers, hidden_size=spec.hidden, seq_len=spec.seq_len)
cfg = ParallelConfig(pp_size=P, dp_size=D, microbatches=B, unit_size=U, stages_per_device=V, microbatch_samples=mbs)
pl = make_placement(cfg, model)
sched = generate(model, cfg, pl)
rt = Runtime(spec, model, cfg, pl, sched, rank=rank, world=world)
tok = synthetic_tokens(1, D, B, mbs, spec.seq_len, spec.vocab)[0, rt.z]
ids = tok[:, :, :-1].reshape(B, -1).contiguous().cuda()
lab = tok[:, :, 1:].reshape(B, -1).contiguous().cuda()
for _ in range(args.warmup):
    rt.step(ids, lab)
rt.join()
torch.cuda.synchronize()
if world > 1:
    dist.barrier()
c0 = counters()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
intra = 0
for _ in range(args.steps):
    intra += rt.step(ids, lab).nccl_bytes_intra
rt.join()
e1.record()
torch.cuda.synchronize()
c1 = counters()
ms = e0.elapsed_time(e1) / args.steps
# stage-boundary P2P sends of this rank per step: one [T, h] bf16 tensor per F whose next
# stage lives on another device and per B whose previous stage does
T, h = spec.tokens_per_microbatch, spec.hidden
sends = 0
for t in sched.per_device[rt.p]:
    if t.kind is TaskKind.F and t.stage < rt.S - 1 and pl.stage_to_device[t.stage + 1] != rt.p:
        sends += 1
    if t.kind is TaskKind.B and t.stage > 0 and pl.stage_to_device[t.stage - 1] != rt.p:
        sends += 1
p2p = sends * T * h * 2
row = {"rank": rank, "p": rt.p, "z": rt.z, "ms_per_step": round(ms, 1),
       "nccl_zero_bytes_per_step": intra // args.steps, "p2p_send_bytes_per_step": p2p}
for n in ("xmit", "rcv", "data_tx", "data_rx"):
    a, b = c0[n], c1[n]
    row[n + "_bytes_per_step"] = None if a is None or b is None else (b - a) // args.steps
row["links_reporting"] = c1["xmit_links"]
tx = row["xmit_bytes_per_step"] if row["xmit_bytes_per_step"] is not None else row["data_tx_bytes_per_step"]
if tx is not None:
    expect = row["nccl_zero_bytes_per_step"] + p2p
    row["tx_over_expected"] = round(tx / expect, 3) if expect else None
    row["tx_GBs_avg_over_step"] = round(tx / (ms / 1e3) / 1e9, 1)
rows = [None] * world
if world > 1:
    dist.all_gather_object(rows, row)
else:
    rows = [row]
if rank == 0:
    print(json.dumps({"config": f"{args.model} P{P}xD{D} B{B} U{U} V{V} b{mbs}", "steps": args.steps,
                      "counter": "NVML NVLINK_COUNT_XMIT/RCV_BYTES summed over links (or THROUGHPUT_DATA_TX/RX)", "ranks": rows}))
