"""Drivers of the C ABI for tests and the benchmark: allocate the flat buffers with torch
(plumbing: device memory, streams, process groups), register them, exchange blobs and run
the training loop of Listing 1 with the shadow loop of Listing 2
 on a side stream.  No arithmetic of the method lives here.

Two group shapes:
  VirtualGroup -- n ranks in this process on one GPU ("virtual ranks"): every rank's calls
                  are issued on ONE stream in rank order, so no kernel waits for another.
  DistRank     -- one process per GPU (torchrun), blobs exchanged with all_gather_object;
                  the collective kernels synchronise across GPUs with in-kernel flags.
"""
from __future__ import annotations

import os

import torch

from . import cm
from . import workloads as W

TORCH_DT = {cm.CM_F32: torch.float32, cm.CM_BF16: torch.bfloat16}


class Rank:
    """One rank's buffers + context.  Construction registers and initialises p_0."""

    def __init__(self, numel, world_size, rank, device, grad_dtype=cm.CM_F32, cap_bytes=W.CAP_BYTES,
                 shm_name="checkmate", ring_depth=2, shadow_place=cm.CM_SHADOW_HOST, flags=0,
                 seed=W.SEED, init_state=True, persist_every=1, overwrite=True):
        self.numel = list(numel)
        # the library refuses to replace a surviving shadow segment unless told to (it is the
        # restore source after a hard kill); these drivers start fresh unless they attach
        if overwrite and not flags & cm.CM_FLAG_ATTACH:
            flags |= cm.CM_FLAG_OVERWRITE
        self.n, self.rank, self.device = world_size, rank, device
        self.grad_dtype, self.cap_bytes, self.seed = grad_dtype, cap_bytes, seed
        self.padded, self.n_buckets, self.tensor_off = cm.plan_buckets(self.numel, grad_dtype, cap_bytes,
                                                                       world_size)
        dev = torch.device("cuda", device)
        # one allocation per flat buffer (CUDA IPC maps whole allocations)
        self.grad = torch.empty(self.padded, dtype=TORCH_DT[grad_dtype], device=dev)
        self.p = torch.empty(self.padded, dtype=torch.float32, device=dev)
        # ZeRO-1 keeps only this rank's shard of the moments (shard-local order)
        mv = self.padded // world_size if flags & cm.CM_FLAG_ZERO1 else self.padded
        self.m = torch.empty(mv, dtype=torch.float32, device=dev)
        self.v = torch.empty(mv, dtype=torch.float32, device=dev)
        self.ctx = cm.Context(world_size, rank, device, ring_depth, shadow_place, shm_name, flags, persist_every)
        self.blob = self.ctx.register_buckets(self.numel, grad_dtype, cap_bytes, self.grad.data_ptr(),
                                              self.p.data_ptr(), self.m.data_ptr(), self.v.data_ptr())
        # these drivers never write gradients on the all-reduce stream between two calls
        # (cm_gen_grads is the library's own launch; DDP hooks produce them on another stream)
        self.ctx.set_param("pdl", 1)
        # A/B switches for tools (collective settings: every rank must use the same value)
        for key in ("lazy_exit", "drain_ctas", "oneshot_max_bytes", "ar_impl", "ar_pipe_blocks", "drain_flush_bytes",
                    "numa_node", "zero1_impl", "shadow_blocks", "pdl", "ar_grid_switch_bytes", "ar_blocks", "persist_queue", "pdl_mode", "n1_copy_engine", "shadow_after_train", "ar_tma_min_bytes",
                    "ar_tma_tile", "ar_tma_stages"):
            val = os.environ.get("CM_" + key.upper())
            if val is not None:
                self.ctx.set_param(key, int(val))
        if init_state:
            with torch.cuda.device(dev):
                s = torch.cuda.current_stream(dev)
                self.ctx.init_state(seed, s)
                s.synchronize()

    def buckets(self):
        return [self.ctx.bucket_info(b) for b in range(self.n_buckets)]


class VirtualGroup:
    """n virtual ranks on one GPU, issued on one stream (no cross-kernel waits)."""

    def __init__(self, numel, world_size, device=0, grad_dtype=cm.CM_F32, cap_bytes=W.CAP_BYTES,
                 shm_name="cmvg", ring_depth=2, shadow_place=cm.CM_SHADOW_HOST, flags=0, seed=W.SEED,
                 gscale=W.GRAD_SCALE, hp=None, persist_every=1, opt="adamw"):
        self.n = world_size
        self.seed, self.gscale = seed, gscale
        self.opt = opt
        self.hp = dict(W.HP_SGD if opt == "sgd" else W.HP)
        if hp:
            self.hp.update(hp)
        self.no_tap = bool(flags & cm.CM_FLAG_NO_TAP)
        self.ranks = [Rank(numel, world_size, r, device, grad_dtype, cap_bytes, shm_name, ring_depth,
                           shadow_place, flags, seed, persist_every=persist_every) for r in range(world_size)]
        blobs = [r.blob for r in self.ranks]
        for r in self.ranks:
            r.ctx.connect(blobs)
        self.dev = torch.device("cuda", device)
        self.stream = torch.cuda.Stream(self.dev, priority=-1)   # training: high priority
        self.side = torch.cuda.Stream(self.dev, priority=0)     # shadow: lowest priority
        self.t = 0
        self.n_buckets = self.ranks[0].n_buckets

    def gen(self, t=None):
        t = self.t if t is None else t
        for r in self.ranks:
            r.ctx.gen_grads(self.seed, t, self.gscale, self.stream)

    def allreduce(self, t=None):
        t = self.t if t is None else t
        for b in range(self.n_buckets):
            for r in self.ranks:
                r.ctx.allreduce_multicast(b, t, self.stream)

    def apply(self, step=None):
        step = self.t + 1 if step is None else step
        for r in self.ranks:
            if self.opt == "sgd":
                r.ctx.apply_step_sgd(step, stream=self.stream, **self.hp)
            else:
                r.ctx.apply_step(step, stream=self.stream, **self.hp)

    def shadow(self, step=None):
        step = self.t + 1 if step is None else step
        for r in self.ranks:
            r.ctx.shadow_apply(step, self.side)

    def step(self, gen=True, shadow=True):
        """One iteration t -> t+1 of Listing 1 (+ Listing 2 on the side stream)."""
        if gen:
            self.gen()
        self.allreduce()
        self.apply()
        if shadow and not self.no_tap:
            self.shadow()
        self.t += 1

    def sync(self):
        self.stream.synchronize()
        self.side.synchronize()

    def finalize(self):
        for r in self.ranks:
            r.ctx.finalize()


class DistRank:
    """This process's rank of a torch.distributed group (one GPU per process)."""

    def __init__(self, numel, grad_dtype=cm.CM_F32, cap_bytes=W.CAP_BYTES, shm_name="cmdist", ring_depth=2,
                 shadow_place=cm.CM_SHADOW_HOST, flags=0, seed=W.SEED, gscale=W.GRAD_SCALE, hp=None,
                 persist_every=1, opt="adamw"):
        import torch.distributed as dist
        self.n = dist.get_world_size()
        self.rank_id = dist.get_rank()
        local = int(os.environ.get("LOCAL_RANK", self.rank_id))
        torch.cuda.set_device(local)
        self.seed, self.gscale = seed, gscale
        self.opt = opt
        self.hp = dict(W.HP_SGD if opt == "sgd" else W.HP)
        if hp:
            self.hp.update(hp)
        self.no_tap = bool(flags & cm.CM_FLAG_NO_TAP)
        self.r = Rank(numel, self.n, self.rank_id, local, grad_dtype, cap_bytes, shm_name, ring_depth,
                      shadow_place, flags, seed, persist_every=persist_every)
        blobs = [None] * self.n
        dist.all_gather_object(blobs, self.r.blob)
        self.r.ctx.connect(blobs)
        self.dev = torch.device("cuda", local)
        self.stream = torch.cuda.Stream(self.dev, priority=-1)   # training: high priority
        self.side = torch.cuda.Stream(self.dev, priority=0)     # shadow: lowest priority
        self.t = 0
        self.n_buckets = self.r.n_buckets

    def step(self, gen=True, shadow=True):
        c = self.r.ctx
        if gen:
            c.gen_grads(self.seed, self.t, self.gscale, self.stream)
        for b in range(self.n_buckets):
            c.allreduce_multicast(b, self.t, self.stream)
        if self.opt == "sgd":
            c.apply_step_sgd(self.t + 1, stream=self.stream, **self.hp)
        else:
            c.apply_step(self.t + 1, stream=self.stream, **self.hp)
        if shadow and not self.no_tap:
            c.shadow_apply(self.t + 1, self.side)
        self.t += 1

    def sync(self):
        self.stream.synchronize()
        self.side.synchronize()
