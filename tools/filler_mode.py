"""C4 with a compute filler (paper_2507_13522_b200/fillerbench.py): Llama-3-8B-shaped DP
iterations, checkpointed vs the no-checkpoint NCCL baseline.

  python -m torch.distributed.run --nproc-per-node N tools/filler_mode.py \
      [--tokens 16384] [--steps 6] [--warmup 2] [--ring-depth 9] [--persist-every 8]
Rank 0 prints one JSON line.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_13522_b200.fillerbench import filler_only_ms, run_arm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=16384, help="tokens per GPU per iteration")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--ring-depth", type=int, default=9)
    ap.add_argument("--persist-every", type=int, default=8)
    ap.add_argument("--shadow", default="host", choices=["host", "device"])
    ap.add_argument("--arms", default="nccl,ours_nockpt,ours_ckpt")
    ap.add_argument("--drain-ctas", type=int, default=-1, help="-1 auto, 0 copy engine, k SM drain CTAs")
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    floor_ms, tflops = filler_only_ms(args, local)
    out = {}
    for arm in args.arms.split(","):
        out[arm] = run_arm(arm, args, rank, world, local)
        torch.cuda.empty_cache()
    if rank == 0:
        res = {"mode": "filler", "workload": "Llama-3-8B-shaped (8,030,261,248 params, 226 buckets), bf16 grads, "
                                             "fp32 master + AdamW state, ZeRO-1; fwd/bwd replaced by bf16 GEMMs "
                                             "of 6*P*T FLOPs",
               "n_gpus": world, "tokens_per_gpu": args.tokens, "shadow": args.shadow,
               "ring_depth": args.ring_depth, "persist_every": args.persist_every, "drain_ctas": args.drain_ctas, "env": {k: v for k, v in os.environ.items() if k.startswith("CM_")},
               "filler_only_ms": floor_ms, "filler_tflops": tflops, **out}
        if "nccl" in out and "ours_ckpt" in out:
            res["ckpt_overhead_pct_vs_nccl"] = (out["ours_ckpt"]["ms_per_iter"] / out["nccl"]["ms_per_iter"] - 1) * 100
        if "ours_nockpt" in out and "ours_ckpt" in out:
            res["ckpt_overhead_pct_vs_ours_nockpt"] = (out["ours_ckpt"]["ms_per_iter"] /
                                                      out["ours_nockpt"]["ms_per_iter"] - 1) * 100
        print(json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
