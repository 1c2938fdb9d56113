"""C4 with a compute filler: Llama-3-8B-shaped data-parallel iterations (bf16 gradients, fp32
master weights and AdamW state, 226 buckets of <= 25 MiB) where the model's forward and
backward are replaced by bf16 GEMMs of the same FLOP count -- 2*P*T forward and 4*P*T
backward for T tokens per GPU, the backward spread over the buckets in the order backward
produces them -- so the checkpoint's cost can be measured against a realistic amount of
compute without the model's weights or data (PAPER.md:495-497 trains
Llama-class models with TorchTitan).

Arms (ZeRO-1 everywhere: the replicated fp32 state of 8B parameters plus a shadow does not
fit next to the filler in one GPU's HBM at n <= 4):
  nccl        -- no checkpoint: per-bucket NCCL reduce_scatter on a comm stream as backward
                 produces it, torch fused AdamW on the own shard, NCCL all_gather of the
                 updated parameters;
  ours_nockpt -- the library's reduce-scatter + sharded AdamW fused with the NVLink
                 parameter all-gather (CM_FLAG_ZERO1 | CM_FLAG_NO_TAP); each bucket's sharded
                 step runs right behind its reduce-scatter on the comm stream (cm_apply_bucket,
                 SURVEY 8 f1), overlapping the rest of the backward (CM_BUCKET_STEP=0: one
                 optimizer kernel after the last bucket, as round 1);
  ours_ckpt   -- the same with the per-iteration checkpoint: tap of every reduced shard,
                 shadow step on a low-priority side stream, host snapshot every K steps.
The filler GEMMs are stock torch (the workload, not the path).
"""
import os

import torch
import torch.distributed as dist

GEMM_N = 4096            # filler GEMM: [T_chunk x 4096] @ [4096 x 4096], bf16
GEMM_ROWS = 8192


def _filler():
    dev = torch.cuda.current_device()
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    a = torch.randn(GEMM_ROWS, GEMM_N, device=dev, dtype=torch.bfloat16, generator=g)
    w = torch.randn(GEMM_N, GEMM_N, device=dev, dtype=torch.bfloat16, generator=g) * 0.01
    out = torch.empty(GEMM_ROWS, GEMM_N, device=dev, dtype=torch.bfloat16)
    flops = 2.0 * GEMM_ROWS * GEMM_N * GEMM_N

    def run(k):
        for _ in range(k):
            torch.mm(a, w, out=out)
    return run, flops


def _schedule(bucket_params, P, tokens, flops):
    """GEMM counts: forward, then one count per bucket (fractions carried so the totals
    match 2PT and 4PT)."""
    fwd = round(2.0 * P * tokens / flops)
    per, carry = [], 0.0
    for pb in bucket_params:
        x = 4.0 * pb * tokens / flops + carry
        k = int(x)
        carry = x - k
        per.append(k)
    return fwd, per


def run_arm(arm, args, rank, world, local):
    from . import cm, harness
    from . import workloads as W
    dev = torch.device("cuda", local)
    numel = W.numels(W.llama3_8b())
    P = sum(numel)
    fill, flops = _filler()
    stream = torch.cuda.current_stream(dev)
    if arm == "nccl":
        R = harness.Rank(numel, world, rank, local, cm.CM_BF16, W.CAP_BYTES, "unused", 2, cm.CM_SHADOW_HOST,
                         cm.CM_FLAG_NO_TAP | cm.CM_FLAG_ZERO1)          # buffers + the input generator
        buckets = R.buckets()
        L = R.padded // world
        gshard = torch.empty(L, dtype=torch.bfloat16, device=dev)
        pshard = torch.empty(L, dtype=torch.float32, device=dev)
        for (o, p, u) in buckets:
            e = p // world
            pshard[o // world:o // world + e].copy_(R.p[o + rank * e:o + (rank + 1) * e])
        step_t = torch.zeros((), dtype=torch.float32, device=dev)
        gscale = torch.full((), float(world), dtype=torch.float32, device=dev)
        comm = torch.cuda.Stream(dev, priority=-1)
        ctx = R.ctx

        def reduce(b, t):
            o, p, u = buckets[b]
            with torch.cuda.stream(comm):
                dist.reduce_scatter_tensor(gshard[o // world:(o + p) // world], R.grad[o:o + p])

        def optimize(t):
            stream.wait_stream(comm)
            step_t.add_(1)
            torch._fused_adamw_([pshard], [gshard.float()], [R.m], [R.v], [], [step_t], amsgrad=False,
                                lr=1e-3, beta1=0.9, beta2=0.999, weight_decay=0.01, eps=1e-8, maximize=False,
                                grad_scale=gscale)
            for (o, p, u) in buckets:
                dist.all_gather_into_tensor(R.p[o:o + p], pshard[o // world:(o + p) // world])
        side = []
        cleanup = lambda: None   # noqa: E731
    else:
        flags = cm.CM_FLAG_ZERO1 | (cm.CM_FLAG_NO_TAP if arm == "ours_nockpt" else 0)
        name = f"cmfb_{os.environ.get('MASTER_PORT', '0')}_{arm}"
        place = cm.CM_SHADOW_DEVICE if args.shadow == "device" else cm.CM_SHADOW_HOST
        D = 2 if arm == "ours_nockpt" else args.ring_depth
        R = harness.DistRank(numel, cm.CM_BF16, W.CAP_BYTES, name, D, place, flags,
                             persist_every=1 if arm == "ours_nockpt" else args.persist_every)
        buckets = R.r.buckets()
        comm = torch.cuda.Stream(dev, priority=-1)
        ctx = R.r.ctx
        if getattr(args, "drain_ctas", -1) != -1:
            ctx.set_param("drain_ctas", args.drain_ctas)

        bucket_step = os.environ.get("CM_BUCKET_STEP", "1") != "0"

        def reduce(b, t):
            ev = torch.cuda.Event()
            ev.record(stream)
            comm.wait_event(ev)
            ctx.allreduce_multicast(b, t, comm)
            if bucket_step:
                ctx.apply_bucket(b, t + 1, stream=comm, **W.HP)

        def optimize(t):
            stream.wait_stream(comm)
            ctx.apply_step(t + 1, stream=stream, **W.HP)
            if arm == "ours_ckpt":
                ctx.shadow_apply(t + 1, R.side)
        side = [R.side]

        def cleanup():
            ok = ctx.verify_ex(cm.CM_VERIFY_ALL, stream)[0] == cm.CM_OK if arm == "ours_ckpt" else None
            ctx.join(stream)
            stream.synchronize()
            ctx.finalize()
            cm.unlink_shadow(name, rank)
            return ok
    fwd, per = _schedule([p for (o, p, u) in buckets], P, args.tokens, flops)

    def iteration(t):
        ctx.gen_grads(0, t, 10, stream)         # gradient production (part of backward)
        fill(fwd)                               # forward
        for b in range(len(buckets)):           # backward: bucket b's grads, then its all-reduce
            fill(per[b])
            reduce(b, t)
        optimize(t)

    for t in range(args.warmup):
        iteration(t)
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for t in range(args.warmup, args.warmup + args.steps):
        iteration(t)
    for s in side + [comm]:
        stream.wait_stream(s)
    if arm != "nccl":
        ctx.join(stream)
    b.record(stream)
    b.synchronize()
    ms = torch.tensor([a.elapsed_time(b) / args.steps], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    drain = ctx.info().drain_ctas if arm != "nccl" else None
    ok = cleanup()
    gemms = fwd + sum(per)
    return {"ms_per_iter": ms.item(), "shadow_bit_identical": ok, "filler_gemms": gemms,
            "filler_tflop": gemms * flops / 1e12, "drain_ctas": drain}


def filler_only_ms(args, local):
    """The filler alone (no communication, no optimizer): the compute floor of an iteration."""
    from . import workloads as W
    numel = W.numels(W.llama3_8b())
    P = sum(numel)
    fill, flops = _filler()
    fwd = round(6.0 * P * args.tokens / flops)
    fill(3)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fill(fwd)
    b.record()
    b.synchronize()
    return a.elapsed_time(b), fwd * flops / (a.elapsed_time(b) * 1e-3) / 1e12
