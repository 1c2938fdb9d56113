"""DDP-style integration of the hot path: a model's parameters and
gradients become views into the library's flat bucket-ordered buffers, and each bucket's
fused all-reduce + tap is launched from backward hooks on a communication stream as soon as
its last gradient is accumulated -- the overlap of gradient computation and
synchronisation the paper's training loop relies on (Listing 1 line
"loss.backward()"; "each model layer points to a specific offset in a
bucket").  The optimizer step is the library's AdamW on the flat fp32 state; the shadow
step runs on a low-priority side stream (Listing 2).

Plumbing only (tensor views, hooks, streams, events); every step of the path runs in the
library's kernels.

bucket_step=True (default): each bucket's optimizer step is launched right behind its
all-reduce on the communication stream (cm_apply_bucket), so the optimizer overlaps the
rest of the backward pass instead of running after it; step() then only finishes the step
(scalar record for the shadow) and launches the shadow step.

A GradProbe (optional) records, for sampled flat indices, every rank's gradients before the
reduce and the state before the step, so a checker can recompute the reduce and the optimizer
step of those elements with the oracle (SURVEY 8.d C2 model-mode parity).
"""
from __future__ import annotations

import os

import torch

from . import cm, harness
from . import workloads as W


class CheckmateDDP:
    def __init__(self, module: torch.nn.Module, device: int, world_size: int = 1, rank: int = 0,
                 cap_bytes: int = W.CAP_BYTES, shm_name: str = "cmddp", ring_depth: int = 16,
                 persist_every: int = 8, shadow_place: int = cm.CM_SHADOW_HOST, flags: int = 0, hp=None,
                 bucket_step: bool = True):
        import torch.distributed as dist
        self.module = module
        self.params = [p for p in module.parameters() if p.requires_grad]
        numel = [p.numel() for p in self.params]
        self.hp = dict(W.HP)
        if hp:
            self.hp.update(hp)
        self.no_tap = bool(flags & (cm.CM_FLAG_NO_TAP | cm.CM_FLAG_NO_SHADOW))
        self.r = harness.Rank(numel, world_size, rank, device, cm.CM_F32, cap_bytes, shm_name, ring_depth,
                              shadow_place, flags, init_state=False, persist_every=persist_every)
        r = self.r
        with torch.no_grad():
            for p, off in zip(self.params, r.tensor_off):
                view = r.p[off:off + p.numel()].view_as(p)
                view.copy_(p.data)
                p.data = view                                  # parameters live in the flat buffer
                p.grad = r.grad[off:off + p.numel()].view_as(p)  # gradients accumulate in place
            # padding of the flat buffers (planner zero-pads every bucket, reading R26)
            used = torch.zeros(r.padded, dtype=torch.bool, device=r.p.device)
            for p, off in zip(self.params, r.tensor_off):
                used[off:off + p.numel()] = True
            r.p.masked_fill_(~used, 0.0)
            r.m.zero_()
            r.v.zero_()
            r.grad.zero_()
        torch.cuda.synchronize(r.p.device)
        if world_size > 1:
            blobs = [None] * world_size
            dist.all_gather_object(blobs, r.blob)
        else:
            blobs = [r.blob]
        r.ctx.connect(blobs)                                   # step-0 shadow snapshot
        self.dev = r.p.device
        self.comm = torch.cuda.Stream(self.dev, priority=-1)
        self.side = torch.cuda.Stream(self.dev, priority=0)
        # bucket of every parameter (by flat offset) and per-bucket pending counts
        buckets = r.buckets()
        self.bucket_of = {}
        self.size = [0] * len(buckets)
        for i, (p, off) in enumerate(zip(self.params, r.tensor_off)):
            for b, (boff, padded, used_n) in enumerate(buckets):
                if boff <= off < boff + padded:
                    self.bucket_of[p] = b
                    self.size[b] += 1
                    break
        self.pending = list(self.size)
        self.t = 0
        self.issued = 0
        self.bucket_step = bucket_step
        # where the per-bucket steps run: right behind the all-reduce on the communication
        # stream (default), or (CM_BUCKET_STREAM=low) on a lowest-priority stream of their own
        # that waits for each bucket's all-reduce, so they yield SMs to the backward pass
        self.opt = None
        if bucket_step and os.environ.get("CM_BUCKET_STREAM", "comm") == "low":
            self.opt = torch.cuda.Stream(self.dev, priority=0)
        self.probe = None
        for p in self.params:
            p.register_post_accumulate_grad_hook(self._hook)

    def _hook(self, p):
        b = self.bucket_of[p]
        self.pending[b] -= 1
        if self.pending[b] == 0:
            if self.probe is not None:                         # (on the producing stream, before
                self.probe.before_reduce(self, b)              # the event: nothing foreign on comm)
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.dev))     # this bucket's grads are written
            self.comm.wait_event(ev)
            self.r.ctx.allreduce_multicast(b, self.t, self.comm)
            if self.bucket_step:
                s = self.comm
                if self.opt is not None:
                    e2 = torch.cuda.Event()
                    e2.record(self.comm)
                    self.opt.wait_event(e2)
                    s = self.opt
                self.r.ctx.apply_bucket(b, self.t + 1, stream=s, **self.hp)
            self.issued += 1

    def zero_grad(self):
        self.r.grad.zero_()
        self.pending = list(self.size)
        self.issued = 0
        if self.probe is not None:
            self.probe.before_step(self)

    def step(self):
        """After loss.backward(): wait for the all-reduces, AdamW, then the shadow step."""
        assert self.issued == len(self.size), "backward did not produce every bucket"
        cur = torch.cuda.current_stream(self.dev)
        cur.wait_stream(self.comm)
        if self.opt is not None:
            cur.wait_stream(self.opt)
        self.r.ctx.apply_step(self.t + 1, stream=cur, **self.hp)   # (remaining buckets +) the step's record
        if self.probe is not None:
            self.probe.after_step(self)
        if not self.no_tap:
            self.r.ctx.shadow_apply(self.t + 1, self.side)
        self.t += 1

    def finalize(self):
        torch.cuda.synchronize(self.dev)
        self.r.ctx.finalize()


class GradProbe:
    """Samples of one iteration for an external parity check (plumbing only: index copies).
    idx: flat indices (sorted) into the registered buffers.  Per iteration it keeps this
    rank's pre-reduce gradients, the pre-step p/m/v and the post-step R, p, m, v at idx."""

    def __init__(self, ddp: CheckmateDDP, idx):
        r = ddp.r
        self.idx = torch.as_tensor(idx, dtype=torch.int64, device=r.p.device)
        buckets = r.buckets()
        self.sel = []
        for off, padded, _ in buckets:
            m = (self.idx >= off) & (self.idx < off + padded)
            self.sel.append(torch.nonzero(m).flatten())
        self.pre_grad = torch.zeros(len(self.idx), dtype=r.grad.dtype, device=r.p.device)
        self.records = []

    def before_step(self, ddp):
        r = ddp.r
        self.cur = {"step": ddp.t + 1, "p": r.p[self.idx].cpu(), "m": r.m[self.idx].cpu(), "v": r.v[self.idx].cpu()}

    def before_reduce(self, ddp, b):
        sel = self.sel[b]
        if len(sel):
            self.pre_grad[sel] = ddp.r.grad[self.idx[sel]]

    def after_step(self, ddp):
        r = ddp.r
        torch.cuda.current_stream(r.p.device).synchronize()
        self.cur.update(grad=self.pre_grad.cpu().clone(), R=r.grad[self.idx].cpu(), p_new=r.p[self.idx].cpu(),
                        m_new=r.m[self.idx].cpu(), v_new=r.v[self.idx].cpu())
        self.records.append(self.cur)
