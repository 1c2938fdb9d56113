"""C5 failure/restore at GPT-2 scale: kill every rank at iteration k (no cleanup: the
processes exit, only the host shadow segments survive), relaunch, attach, restore from the
shadow, continue 100 iterations, and compare sampled elements of every rank's state with
the oracle's uninterrupted trajectories, bit for bit.

  python -m torch.distributed.run --nproc-per-node N tools/restore_bench.py phase1 <name> [k] [more] [point]
  python -m torch.distributed.run --nproc-per-node N tools/restore_bench.py phase2kill <name> [k] [more] [delay_s]
  python -m torch.distributed.run --nproc-per-node N tools/restore_bench.py phase2 <name> [k] [more]
Kill points of phase 1: "step" (after k whole iterations, their shadow
and drain work still in flight), "before_rs" (k whole iterations, then iteration k's
gradients produced, no all-reduce issued), "after_ar" (k whole iterations, then iteration
k's gradients and all-reduces + taps issued, the optimizer step never reached),
"mid_shadow" (k whole iterations with k a multiple of K = 8, killed 5 ms after the last
one was issued: its shadow step and the persist of the 1.5 GB snapshot are in flight).  phase2kill
attaches, starts cm_restore and SIGKILLs itself after delay_s (a kill mid-restore, possibly
mid-persist of the rolled-forward snapshot); phase 2 must still restore.
Rank 0 of phase 2 prints one JSON line (restore wall time, restored step, bit-exactness).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_13522_b200 import cm, harness  # noqa: E402
from paper_2507_13522_b200 import workloads as W  # noqa: E402


def main():
    phase, name = sys.argv[1], sys.argv[2]
    k = int(sys.argv[3]) if len(sys.argv) > 3 else 7
    more = int(sys.argv[4]) if len(sys.argv) > 4 else 100
    extra = sys.argv[5] if len(sys.argv) > 5 else None
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, n = dist.get_rank(), dist.get_world_size()
    llama = os.environ.get("CM_RESTORE_WORKLOAD", "gpt2") == "llama8b"
    # GPT-2 (fp32, replicated AdamW, K=8, D=16) or the Llama-3-8B shape (bf16 grads, ZeRO-1:
    # the replicated fp32 state of 8B parameters does not fit next to the shadow at n <= 4)
    numel = W.numels(W.llama3_8b()) if llama else W.numels(W.gpt2_small())
    dtype = cm.CM_BF16 if llama else cm.CM_F32
    D, K = (9, 8) if llama else (16, 8)
    flags = cm.CM_FLAG_ATTACH if phase in ("phase2", "phase2kill") else 0
    if llama:
        flags |= cm.CM_FLAG_ZERO1
    R = harness.DistRank(numel, dtype, W.CAP_BYTES, name, D, cm.CM_SHADOW_HOST, flags, persist_every=K)
    if phase == "phase1":
        for _ in range(k):
            R.step()
        c = R.r.ctx
        if extra in ("after_ar", "before_rs"):
            c.gen_grads(R.seed, R.t, R.gscale, R.stream)
            if extra == "after_ar":
                for b in range(R.n_buckets):
                    c.allreduce_multicast(b, R.t, R.stream)
        if extra == "mid_shadow":
            time.sleep(0.005)                 # the last shadow step + snapshot persist in flight
            os._exit(0)
        # die with work still in flight (no stream sync, no finalize): whatever the GPUs did
        # not finish is lost; only the host shadow segments in /dev/shm survive
        dist.barrier()
        os._exit(0)
    # phase 2: fresh processes, garbage training state
    torch.cuda.synchronize()
    R.r.p.fill_(float("nan"))
    R.r.m.fill_(float("nan"))
    R.r.v.fill_(float("nan"))
    torch.cuda.synchronize()
    dist.barrier()
    if phase == "phase2kill":
        import signal
        import threading
        delay = float(extra) if extra else 0.02
        threading.Timer(delay, lambda: os.kill(os.getpid(), signal.SIGKILL)).start()
        R.r.ctx.restore(R.stream)
        torch.cuda.synchronize()
        time.sleep(10)                      # the timer fires (restore was faster than delay)
    t0 = time.perf_counter()
    I = R.r.ctx.restore(R.stream)
    torch.cuda.synchronize()
    restore_s = time.perf_counter() - t0
    R.t = I
    for _ in range(more):
        R.step()
    R.sync()
    ok_shadow = R.r.ctx.verify_ex(cm.CM_VERIFY_ALL, R.stream)[0] == cm.CM_OK
    # sampled bitwise comparison with the oracle's uninterrupted trajectories
    from oracle import oracle as O
    plan = O.Plan(numel, W.CAP_BYTES, 2 if llama else 4, n)
    rng = np.random.default_rng(rank)
    idx = np.sort(rng.choice(plan.total, 1 << 14, replace=False)).astype(np.int64)
    bi = np.searchsorted(plan.bucket_off, idx, side="right") - 1
    used = ((idx - plan.bucket_off[bi]) < plan.bucket_used[bi]).astype(np.uint8)
    p, m, v, Rl = O.run_sample(W.SEED, n, O.BF16 if llama else O.F32, W.GRAD_SCALE, I + more, idx, used,
                               lr=W.HP["lr"], b1=W.HP["beta1"], b2=W.HP["beta2"], eps=W.HP["eps"],
                               wd=W.HP["weight_decay"])
    ti = torch.from_numpy(idx).to(R.r.p.device)
    same = np.array_equal(R.r.p[ti].cpu().numpy().view(np.uint32), p.view(np.uint32))
    if llama:     # m, v are shard-local: this rank's shard of the sampled elements
        e = plan.bucket_padded[bi] // n
        local = idx - plan.bucket_off[bi] - rank * e
        mine = (local >= 0) & (local < e)
        tj = torch.from_numpy((plan.bucket_off[bi] // n + local)[mine]).to(R.r.m.device)
        same = same and np.array_equal(R.r.m[tj].cpu().numpy().view(np.uint32), m[mine].view(np.uint32)) \
            and np.array_equal(R.r.v[tj].cpu().numpy().view(np.uint32), v[mine].view(np.uint32))
    else:
        same = same and all(np.array_equal(a[ti].cpu().numpy().view(np.uint32), b.view(np.uint32))
                            for a, b in ((R.r.m, m), (R.r.v, v)))
    res = torch.tensor([restore_s, float(same and ok_shadow)], dtype=torch.float64, device=R.r.p.device)
    dist.all_reduce(res, op=dist.ReduceOp.MAX)
    ok_all = torch.tensor([float(same and ok_shadow)], dtype=torch.float64, device=R.r.p.device)
    dist.all_reduce(ok_all, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(json.dumps({"workload": "llama8b (ZeRO-1, bf16 grads)" if llama else "gpt2", "n": n,
                          "restore_bytes_h2d_per_gpu": int(12 * plan.total / n),
                          "killed_after_iterations": k, "kill_point": os.environ.get("CM_KILL_POINT", "step"),
                          "restored_step": I, "restore_s_max_over_ranks": res[0].item(),
                          "continued_iterations": more, "bit_exact_vs_oracle_and_shadow": bool(ok_all.item() == 1.0),
                          "sampled_elements_per_rank": int(len(idx)), "persist_every": K, "ring_depth": D}),
              flush=True)
    dist.barrier()
    R.r.ctx.finalize()
    cm.unlink_shadow(name, rank)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
