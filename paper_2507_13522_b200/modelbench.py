"""GPT-2 model mode (C2): data-parallel training iterations of a real model (random init,
random tokens, bf16 autocast, seq 1024) with the per-iteration checkpoint (CheckmateDDP)
vs the no-checkpoint baseline (torch DDP over NCCL + torch fused AdamW).  Used by
bench.py and tools/model_mode.py.  The model's fwd/bwd is stock PyTorch (the workload, not
the path); the all-reduce + tap, AdamW and shadow are the library's kernels.
"""
import os

import torch
import torch.distributed as dist


def make_model(seed):
    from transformers import GPT2Config, GPT2LMHeadModel
    torch.manual_seed(seed)
    cfg = GPT2Config()
    cfg._attn_implementation = "sdpa"
    return GPT2LMHeadModel(cfg)


def run_arm(arm, args, rank, world, local):
    from . import cm
    from .ddp import CheckmateDDP
    dev = torch.device("cuda", local)
    # the step's tail after backward: an event on the compute stream when backward's kernels
    # are done (for torch DDP: after its all-reduce wait at the end of backward) and one when
    # the step is done (ours: after the library step on the compute stream, which waits for the
    # communication stream's all-reduces and per-bucket optimizer steps)
    marks = {"on": False, "pairs": [], "cur": None}

    def mark(k):
        if not marks["on"]:
            return
        e = torch.cuda.Event(enable_timing=True)
        e.record(torch.cuda.current_stream(dev))
        if k == 0:
            marks["cur"] = e
        else:
            marks["pairs"].append((marks["cur"], e))
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
            mark(0)
            opt.step()
            mark(1)
        streams = []
        cleanup = lambda: None   # noqa: E731
    else:
        flags = cm.CM_FLAG_NO_TAP if arm in ("ours_nockpt", "nockpt_d2hload", "nockpt_d2hpaced") else (
            {"ce": cm.CM_FLAG_TAP_COPYENGINE, "direct": cm.CM_FLAG_TAP_DIRECT}.get(args.tap, 0))
        if arm in ("ours_tap_only", "ours_tap_nodrain"):   # tap into the ring, no shadow replica
            flags |= cm.CM_FLAG_NO_SHADOW
        if getattr(args, "zero1", False):
            flags |= cm.CM_FLAG_ZERO1
        name = f"cmmm_{os.environ.get('MASTER_PORT', '0')}_{arm}"
        # per-bucket optimizer steps behind each bucket's all-reduce (default; CM_BUCKET_STEP=0:
        # one optimizer kernel after backward, the A/B arm)
        cd = CheckmateDDP(model, local, world, rank, shm_name=name, ring_depth=args.ring_depth,
                          persist_every=args.persist_every, flags=flags,
                          bucket_step=os.environ.get("CM_BUCKET_STEP", "1") != "0")
        if getattr(args, "drain_ctas", -1) != -1:   # override the library's auto drain policy
            cd.r.ctx.set_param("drain_ctas", args.drain_ctas)
        if arm == "ours_tap_nodrain":               # cost decomposition: staging stores, no D2H
            cd.r.ctx.set_param("ablate_no_drain", 1)
        load = None
        pace = None
        if arm == "nockpt_d2hpaced":                # the same bytes, released in small chunks
            nb = cd.r.padded * 4 // world           # from forward pre-hooks (one per module)
            src = torch.empty(nb, dtype=torch.uint8, device=dev)
            dst = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
            ls = torch.cuda.Stream(dev)
            mods = [m for m in model.modules() if len(list(m.children())) == 0]
            cs = (nb + len(mods) - 1) // len(mods)
            pace = {"i": 0}

            def pre_hook(mod, inp):
                j = pace["i"]
                pace["i"] += 1
                lo = j * cs
                if lo < nb:
                    ls.wait_stream(torch.cuda.current_stream())
                    with torch.cuda.stream(ls):
                        dst[lo:lo + cs].copy_(src[lo:lo + cs], non_blocking=True)
            for mm in mods:
                mm.register_forward_pre_hook(pre_hook)
            load = (None, None, ls)
        if arm == "nockpt_d2hload":                 # cost decomposition: the tap's D2H bytes
            nb = cd.r.padded * 4 // world           # (S/n per iteration) as a plain copy-engine
            load = (torch.empty(nb, dtype=torch.uint8, device=dev),  # load on its own stream,
                    torch.empty(nb, dtype=torch.uint8, pin_memory=True),   # no tap, no shadow
                    torch.cuda.Stream(dev))

        def it(i):
            cd.zero_grad()
            if pace is not None:
                pace["i"] = 0
            if load is not None and pace is None:
                load[2].wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(load[2]):
                    load[1].copy_(load[0], non_blocking=True)
            with torch.autocast("cuda", dtype=torch.bfloat16):
                loss = model(tokens[i], labels=tokens[i]).loss
            loss.backward()
            mark(0)
            cd.step()
            mark(1)
        streams = [cd.comm, cd.side] + ([load[2]] if load is not None else [])

        def cleanup():
            full = not (flags & (cm.CM_FLAG_NO_TAP | cm.CM_FLAG_NO_SHADOW))
            ok = cd.r.ctx.verify_ex(cm.CM_VERIFY_ALL, torch.cuda.current_stream())[0] == cm.CM_OK if full else None
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
    lags = []
    has_shadow = arm not in ("nccl",) and not (flags & (cm.CM_FLAG_NO_TAP | cm.CM_FLAG_NO_SHADOW))
    marks["on"] = True
    for i in range(args.warmup, args.warmup + args.steps):
        it(i)
        if has_shadow:   # training steps issued minus the step the shadow has published
            lags.append(cd.t - cd.r.ctx.info().shadow_step)
    for s in streams:
        cur.wait_stream(s)
    b.record(cur)
    b.synchronize()
    ms = torch.tensor([a.elapsed_time(b) / args.steps], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    drain = cd.r.ctx.info().drain_ctas if arm not in ("nccl",) else None
    ok = cleanup()
    del model
    torch.cuda.empty_cache()
    tail = sum(a.elapsed_time(b) for a, b in marks["pairs"]) / max(1, len(marks["pairs"]))
    out = {"ms_per_iter": ms.item(), "shadow_bit_identical": ok, "drain_ctas": drain,
           "tail_after_backward_ms": tail}
    if lags:
        out["shadow_lag_iters"] = {"max": max(lags), "mean": sum(lags) / len(lags),
                                   "what": "steps the host has issued minus the step the shadow published, "
                                           "sampled after each timed iteration is issued (rank 0)"}
    return out


