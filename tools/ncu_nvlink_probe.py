"""ncu target for NVLink counters of the all-reduce kernels: ONE process drives N GPUs (ranks
in-process on devices 0..N-1, peer access over NVLink) with the cross-GPU barriers off
(profiling only), so ncu can serialise the kernels without a kernel waiting for a peer that
ncu holds back.  Each rank's kernel still pulls its shard from every peer and pushes the
result to every peer over NVLink: its nvlrx/nvltx bytes are the per-GPU traffic of one
two-shot all-reduce launch (the values computed are meaningless without the barriers).

  ncu --metrics ... python tools/ncu_nvlink_probe.py [--n 2] [--impl -1|0|2] [--zero1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2507_13522_b200 import cm, harness  # noqa: E402
from paper_2507_13522_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2)
ap.add_argument("--impl", type=int, default=-1)
ap.add_argument("--zero1", action="store_true")
a = ap.parse_args()
numel = W.numels(W.gpt2_small())
flags = cm.CM_FLAG_NO_TAP | (cm.CM_FLAG_ZERO1 if a.zero1 else 0)
ranks = []
for r in range(a.n):
    torch.cuda.set_device(r)
    rk = harness.Rank(numel, a.n, r, r, cm.CM_F32, W.CAP_BYTES, "unused", 2, cm.CM_SHADOW_HOST, flags)
    rk.ctx.set_param("force_no_barriers", 1)
    rk.ctx.set_param("ar_impl", a.impl)
    ranks.append(rk)
blobs = [rk.blob for rk in ranks]
for rk in ranks:
    torch.cuda.set_device(rk.device)
    rk.ctx.connect(blobs)
streams = [torch.cuda.Stream(torch.device("cuda", rk.device)) for rk in ranks]
# (the library enqueues on the calling thread's current device: set it per rank)
for t in range(2):
    for rk, s in zip(ranks, streams):
        torch.cuda.set_device(rk.device)
        rk.ctx.gen_grads(0, t, 10, s)
    for b in range(ranks[0].n_buckets):
        for rk, s in zip(ranks, streams):
            torch.cuda.set_device(rk.device)
            rk.ctx.allreduce_multicast(b, t, s)
    for rk, s in zip(ranks, streams):
        torch.cuda.set_device(rk.device)
        rk.ctx.apply_step(t + 1, stream=s, **W.HP)
    for s in streams:
        s.synchronize()
print("probe ok", a.n, ranks[0].n_buckets)
for rk in ranks:
    torch.cuda.set_device(rk.device)
    rk.ctx.finalize()
