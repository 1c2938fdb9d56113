"""Small, deterministic target for ncu: a few iterations of the full hot path.

  python tools/prof_target.py [--n N] [--steps K] [--dtype f32|bf16] [--shadow host|device]
N virtual ranks on one GPU (no cross-kernel waits, safe under ncu's kernel replay).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2507_13522_b200 import cm, harness  # noqa: E402
from paper_2507_13522_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--shadow", default="host")
ap.add_argument("--opt", default="adamw", choices=["adamw", "sgd"])
ap.add_argument("--drain-ctas", type=int, default=-1, help="force the SM drain (k CTAs) for profiling it")
ap.add_argument("--ring-depth", type=int, default=2)
ap.add_argument("--persist-every", type=int, default=1)
a = ap.parse_args()
dtype = cm.CM_F32 if a.dtype == "f32" else cm.CM_BF16
name = f"cmprof{os.getpid()}"
g = harness.VirtualGroup(W.numels(W.gpt2_small()), a.n, 0, dtype, W.CAP_BYTES, name, a.ring_depth,
                         cm.CM_SHADOW_HOST if a.shadow == "host" else cm.CM_SHADOW_DEVICE, opt=a.opt,
                         persist_every=a.persist_every)
if a.drain_ctas >= 0:
    for r in g.ranks:
        r.ctx.set_param("drain_ctas", a.drain_ctas)
for _ in range(a.steps):
    g.step()
g.sync()
bad = [r.ctx.verify(g.stream) for r in g.ranks]
g.finalize()
for r in range(a.n):
    cm.unlink_shadow(name, r)
assert all(b == -1 for b in bad), bad
print("prof_target ok", a.n, a.steps)
