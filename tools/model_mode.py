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


def make_model(seed):
    from transformers import GPT2Config, GPT2LMHeadModel
    torch.manual_seed(seed)
    cfg = GPT2Config()
    cfg._attn_implementation = "sdpa"
    return GPT2LMHeadModel(cfg)


def run_arm(arm, args, rank, world, local):
    from paper_2507_13522_b200 import cm
    from paper_2507_13522_b200.ddp import CheckmateDDP
    dev = torch.device("cuda", local)
    model = make_model(0).to(dev)
    model.train()
    g = torch.Generator(device=dev)
    g.manual_seed(1000 + rank)
    tokens = torch.randint(0, 50257, (args.steps + args.warmup, args.micro_batch, 1024), device=dev, generator=g)
    if arm == "nccl":
        ddp = torch.nn.parallel.DistributedDataParallel(model, device_ids=[local], bucket_cap_mb=25,
                                                        gradient_as_bucket_view=True)
        opt = torch.optim.AdamW(model.parameters(), lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01,
                                fused=True)

        def it(i):
            opt.zero_grad(set_to_none=False)
            with torch.autocast("cuda", dtype=torch.bfloat16):
                loss = ddp(tokens[i], labels=tokens[i]).loss
            loss.backward()
            opt.step()
        streams = []
        cleanup = lambda: None   # noqa: E731
    else:
        flags = cm.CM_FLAG_NO_TAP if arm == "ours_nockpt" else (
            {"ce": cm.CM_FLAG_TAP_COPYENGINE, "direct": cm.CM_FLAG_TAP_DIRECT}.get(args.tap, 0))
        if arm == "ours_tap_only":                  # tap into the ring, no shadow replica
            flags |= cm.CM_FLAG_NO_SHADOW
        name = f"cmmm_{os.environ.get('MASTER_PORT', '0')}_{arm}"
        cd = CheckmateDDP(model, local, world, rank, shm_name=name, ring_depth=args.ring_depth,
                          persist_every=args.persist_every, flags=flags)

        def it(i):
            cd.zero_grad()
            with torch.autocast("cuda", dtype=torch.bfloat16):
                loss = model(tokens[i], labels=tokens[i]).loss
            loss.backward()
            cd.step()
        streams = [cd.comm, cd.side]

        def cleanup():
            full = not (flags & (cm.CM_FLAG_NO_TAP | cm.CM_FLAG_NO_SHADOW))
            ok = cd.r.ctx.verify(torch.cuda.current_stream()) == -1 if full else None
            cd.finalize()
            cm.unlink_shadow(name, rank)
            return ok
    for i in range(args.warmup):
        it(i)
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    a.record(cur)
    for i in range(args.warmup, args.warmup + args.steps):
        it(i)
    for s in streams:
        cur.wait_stream(s)
    b.record(cur)
    b.synchronize()
    ms = torch.tensor([a.elapsed_time(b) / args.steps], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ok = cleanup()
    del model
    torch.cuda.empty_cache()
    return {"ms_per_iter": ms.item(), "shadow_bit_identical": ok}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--micro-batch", type=int, default=16)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--ring-depth", type=int, default=16)
    ap.add_argument("--persist-every", type=int, default=8)
    ap.add_argument("--arms", default="nccl,ours_nockpt,ours_ckpt")
    ap.add_argument("--tap", default="staged", choices=["staged", "direct", "ce"])
    args = ap.parse_args()
    rank, world, local = setup()
    out = {}
    for arm in args.arms.split(","):
        out[arm] = run_arm(arm, args, rank, world, local)
    if rank == 0:
        res = {"mode": "model", "model": "GPT-2 small (124M), random init, random tokens", "n_gpus": world,
               "micro_batch": args.micro_batch, "seq_len": 1024, "autocast": "bf16", "persist_every":
               args.persist_every, "ring_depth": args.ring_depth, "tap": args.tap, **out}
        if "nccl" in out and "ours_ckpt" in out:
            res["ckpt_overhead_pct_vs_nccl"] = (out["ours_ckpt"]["ms_per_iter"] / out["nccl"]["ms_per_iter"] - 1) * 100
        if "ours_nockpt" in out and "ours_ckpt" in out:
            res["ckpt_overhead_pct_vs_ours_nockpt"] = (out["ours_ckpt"]["ms_per_iter"] /
                                                       out["ours_nockpt"]["ms_per_iter"] - 1) * 100
        print(json.dumps(res), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
