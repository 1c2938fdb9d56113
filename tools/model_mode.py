"""C2 model mode: GPT-2 small (random init, random tokens, bf16 autocast, seq 1024) data-
parallel training, iteration time with the per-iteration checkpoint (CheckmateDDP: fused
all-reduce + tap from backward hooks, library AdamW, shadow on a side stream) vs the
no-checkpoint baseline (torch DDP over NCCL + torch fused AdamW), same model and batch.

  python tools/model_mode.py [--micro-batch 16] [--steps 20] [--warmup 5]
  python -m torch.distributed.run --nproc-per-node N tools/model_mode.py ...
Rank 0 prints one JSON line.
"""
import argparse
import json
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_13522_b200.modelbench import run_arm  # noqa: E402


def setup():
    if "RANK" not in os.environ:
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=str(s.getsockname()[1]))
        s.close()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return dist.get_rank(), dist.get_world_size(), local


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--micro-batch", type=int, default=16)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--ring-depth", type=int, default=16)
    ap.add_argument("--persist-every", type=int, default=8)
    ap.add_argument("--arms", default="nccl,ours_nockpt,ours_ckpt")
    ap.add_argument("--tap", default="staged", choices=["staged", "direct", "ce"])
    ap.add_argument("--zero1", action="store_true")
    ap.add_argument("--drain-ctas", type=int, default=-1,
                    help="tap drain / persist D2H: -1 library auto policy, 0 copy engine, k > 0 a k-CTA "
                         "SM drain kernel")
    args = ap.parse_args()
    rank, world, local = setup()
    out = {}
    for arm in args.arms.split(","):
        out[arm] = run_arm(arm, args, rank, world, local)
    if rank == 0:
        res = {"mode": "model", "model": "GPT-2 small (124M), random init, random tokens", "n_gpus": world,
               "micro_batch": args.micro_batch, "seq_len": 1024, "autocast": "bf16", "persist_every":
               args.persist_every, "ring_depth": args.ring_depth, "tap": args.tap, "zero1": args.zero1,
               "drain_ctas": args.drain_ctas,
               "env": {k: v for k, v in os.environ.items() if k.startswith("CM_")}, **out}
        if "nccl" in out and "ours_ckpt" in out:
            res["ckpt_overhead_pct_vs_nccl"] = (out["ours_ckpt"]["ms_per_iter"] / out["nccl"]["ms_per_iter"] - 1) * 100
        if "ours_nockpt" in out and "ours_ckpt" in out:
            res["ckpt_overhead_pct_vs_ours_nockpt"] = (out["ours_ckpt"]["ms_per_iter"] /
                                                       out["ours_nockpt"]["ms_per_iter"] - 1) * 100
        print(json.dumps(res), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
