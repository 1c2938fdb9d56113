"""Multi-process target for ncu NVLink counters: GPT-2-shaped buckets (17, fp32), N ranks,
a few checkpointed iterations (staged tap, host shadow), optionally ZeRO-1.

  python -m torch.distributed.run --nproc-per-node N tools/ncu_target_mp.py [--steps 2] [--zero1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_13522_b200 import cm, harness  # noqa: E402
from paper_2507_13522_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--zero1", action="store_true")
a = ap.parse_args()
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
name = f"cmncu_{os.environ.get('MASTER_PORT', '0')}"
R = harness.DistRank(W.numels(W.gpt2_small()), cm.CM_F32, W.CAP_BYTES, name, 3, cm.CM_SHADOW_HOST,
                     cm.CM_FLAG_ZERO1 if a.zero1 else 0, persist_every=2)
for _ in range(a.steps):
    R.step()
R.sync()
st = R.r.ctx.verify_ex(cm.CM_VERIFY_ALL, R.stream)
dist.barrier()
R.r.ctx.finalize()
cm.unlink_shadow(name, dist.get_rank())
print(f"rank {dist.get_rank()}: ncu target ok {st}", flush=True)
dist.destroy_process_group()
