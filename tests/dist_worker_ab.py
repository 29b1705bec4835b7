"""One rank of an A/B determinism check under torchrun (or alone at world 1): the same
ZeroPP steps run twice in fresh runtimes, with the early optimizer on and off
(Runtime(early_opt=...)); fp32 master shards and bf16 shards must be bit-identical -- the early
(chunked, overlapped) AdamW and the per-stage AG gating only reorder work, and every
gradient path is deterministic (no fp32 atomics).  The reported loss is an fp32 atomic
sum over token rows, so it is compared to 1e-6 relative.

With arm ``notail`` (8th argument) arm B keeps the early optimizer but runs each step's tail
serially (Runtime(overlap_tail=False)) instead of overlapping it with the next step.

usage: torchrun --nproc-per-node P*D dist_worker_ab.py P D B U V STEPS OUTDIR [noearly|notail]
"""

import os

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import sys

import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

from engine_harness import run_engine_step  # noqa: E402
from paper_2402_03791_b200.engine import GPTSpec  # noqa: E402


def run(early: str, P, D, B, U, V, steps, rank, world, tail: bool = True):
    rt, _, _, res = run_engine_step(GPTSpec.tiny(), P, D, B, U, V, rank=rank, world=world, steps=steps,
                                    timeline=False, rt_kw={"early_opt": early == "1", "overlap_tail": tail})
    assert rt.early_opt == (early == "1")
    losses = [r.loss_sum.item() for r in res]
    state = {s: (st.master.cpu(), st.shard_bf16.cpu()) for s, st in rt.stages.items()}
    del rt
    torch.cuda.synchronize()
    return losses, state


def main():
    P, D, B, U, V, steps = (int(x) for x in sys.argv[1:7])
    out = sys.argv[7]
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    if world > 1:
        dist.init_process_group("gloo")
    msg = "OK"
    try:
        arm = sys.argv[8] if len(sys.argv) > 8 else "noearly"
        la, sa = run("1", P, D, B, U, V, steps, rank, world)
        if arm == "notail":
            lb, sb = run("1", P, D, B, U, V, steps, rank, world, tail=False)
        else:
            lb, sb = run("0", P, D, B, U, V, steps, rank, world)
        fails = []
        if any(abs(a - b) > 1e-6 * abs(b) for a, b in zip(la, lb)):
            fails.append(f"losses differ: {la} vs {lb}")
        for s in sa:
            if not torch.equal(sa[s][0], sb[s][0]):
                fails.append(f"stage {s} master differs")
            if not torch.equal(sa[s][1], sb[s][1]):
                fails.append(f"stage {s} bf16 shard differs")
        if fails:
            msg = "FAIL " + "; ".join(fails)
        else:
            msg = f"OK losses={la}"
    except Exception:
        import traceback
        msg = "FAIL " + traceback.format_exc()
    with open(os.path.join(out, f"rank{rank}.txt"), "w") as f:
        f.write(msg)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    sys.exit(0 if msg.startswith("OK") else 1)


if __name__ == "__main__":
    main()
