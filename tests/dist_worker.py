"""One rank of a multi-GPU ZeroPP step under torchrun; compares its shards with the oracle.

usage: torchrun --nproc-per-node n*P*D dist_worker.py P D B U V OUTDIR [n MODE [RS_WIRE]]

n = inter_node_dp replicas emulated on one box, MODE = dp_outer | zero1_outer.
"""

import os

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")  # see zpp_preload_kernels
import sys

import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

from engine_harness import LOSS_RTOL, compare_shards, oracle_for, run_engine_step  # noqa: E402
from paper_2402_03791_b200 import HybridMode  # noqa: E402
from paper_2402_03791_b200.engine import GPTSpec  # noqa: E402


def main():
    P, D, B, U, V = (int(x) for x in sys.argv[1:6])
    out = sys.argv[6]
    n = int(sys.argv[7]) if len(sys.argv) > 7 else 1
    mode = sys.argv[8] if len(sys.argv) > 8 else "dp_outer"
    rs_wire = sys.argv[9] if len(sys.argv) > 9 else "bf16"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    spec = GPTSpec.tiny()
    msg = "OK"
    try:
        rt, (model, cfg, pl, sched), tokens, res = run_engine_step(spec, P, D, B, U, V, rank=rank, world=world,
                                                                    inter_node_dp=n,
                                                                    hybrid_mode=HybridMode(mode),
                                                                    rt_kw={"rs_wire": rs_wire})
        loss_sum = torch.tensor([res[0].loss_sum.item()])
        dist.all_reduce(loss_sum)
        loss = loss_sum.item() / (n * D * B * spec.tokens_per_microbatch)
        loss_o, grads_o, new_o = oracle_for(spec, cfg, pl, tokens[0])
        fails = compare_shards(spec, cfg, pl, rt, grads_o, new_o)
        sim = res[0].sim  # whole-job measured timeline gathered from every pipeline rank
        if sim is None or set(sim.task_times) != set(sched.tasks()) or sim.extras.get("partial"):
            fails.append("measured timeline does not cover every device's tasks")
        elif not all(0 < b <= sim.makespan for b in sim.per_device_busy):
            fails.append(f"measured busy/makespan inconsistent: {sim.per_device_busy} / {sim.makespan}")
        from paper_2402_03791_b200.engine.model import nccl_bytes_per_step
        want = nccl_bytes_per_step(spec, cfg, pl, sched, rt.p, rs_wire=rs_wire)
        got = (res[0].nccl_bytes_intra, res[0].nccl_bytes_inter)
        if got != want:
            fails.append(f"NCCL bytes {got} != planned {want}")
        if abs(loss - loss_o) / loss_o > LOSS_RTOL:
            fails.append(f"loss {loss} vs oracle {loss_o}")
        if fails:
            msg = "FAIL " + "; ".join(fails)
        else:
            msg = f"OK loss={loss:.5f} oracle={loss_o:.5f} step_ms={res[0].step_ms:.2f}"
    except Exception as exc:  # report, then fail the rank
        import traceback
        msg = "FAIL " + traceback.format_exc()
    with open(os.path.join(out, f"rank{rank}.txt"), "w") as f:
        f.write(msg)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if msg.startswith("OK") else 1)


if __name__ == "__main__":
    main()
