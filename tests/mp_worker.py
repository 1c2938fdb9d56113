"""Worker for the multi-process GPU tests (one process per GPU, launched by
torch.distributed.run from tests/test_gpu_multiproc.py).  Each rank runs the hot path over
real NVLink peer memory and checks its own state bit-for-bit against the oracle.

  python -m torch.distributed.run --nproc-per-node N tests/mp_worker.py <mode> <name>
modes: parity_f32, parity_bf16, parity_zero1, parity_sgd, parity_oneshot, parity_oneshot_bf16,
       parity_oneshot_direct, parity_nvls, parity_nvls_bf16, parity_zero1_oneshot, restore_soft, hardkill_phase1, hardkill_phase2
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2507_13522_b200 import cm, harness  # noqa: E402
from paper_2507_13522_b200 import workloads as W  # noqa: E402

HP_O = dict(lr=W.HP["lr"], b1=W.HP["beta1"], b2=W.HP["beta2"], eps=W.HP["eps"], wd=W.HP["weight_decay"])


def bits(a):
    a = np.asarray(a)
    return a.view(np.uint32) if a.dtype == np.float32 else a


def t2np(t):
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def shard_of(flat, plan, rank):
    n = plan.world_size
    return np.concatenate([flat[o + rank * (p // n): o + (rank + 1) * (p // n)]
                           for o, p in zip(plan.bucket_off, plan.bucket_padded)])


def check(R, ref, what, plan=None):
    r = R.r
    if plan is not None:   # ZeRO-1: full p everywhere, shard-local m/v, no gradient all-gather
        np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p), err_msg=f"{what}: p rank {R.rank_id}")
        np.testing.assert_array_equal(bits(t2np(r.m)), bits(shard_of(ref.m, plan, R.rank_id)))
        np.testing.assert_array_equal(bits(t2np(r.v)), bits(shard_of(ref.v, plan, R.rank_id)))
        assert r.ctx.verify(R.stream) == -1, f"{what}: shadow != train on rank {R.rank_id}"
        return
    np.testing.assert_array_equal(bits(t2np(r.grad)), bits(ref.R), err_msg=f"{what}: R rank {R.rank_id}")
    for nm, a, b in (("p", r.p, ref.p), ("m", r.m, ref.m), ("v", r.v, ref.v)):
        np.testing.assert_array_equal(bits(t2np(a)), bits(b), err_msg=f"{what}: {nm} rank {R.rank_id}")
    assert r.ctx.verify(R.stream) == -1, f"{what}: shadow != train on rank {R.rank_id}"


def llama_full_zero1(name):
    """BASELINE.json configs[3] at full size: Llama-3-8B-shaped (8.03 B params, 226 buckets,
    bf16 grads) ZeRO-1 with the host shadow, 3 iterations; every rank's full p and its
    shard-local m, v compared with the oracle's per-element trajectories on sampled indices
    (PAPER.md:306-308 element independence), plus the shadow verify."""
    n, rank = dist.get_world_size(), dist.get_rank()
    numel = W.numels(W.llama3_8b())
    R = harness.DistRank(numel, cm.CM_BF16, W.CAP_BYTES, name, 4, cm.CM_SHADOW_HOST, cm.CM_FLAG_ZERO1,
                         persist_every=2)
    steps = 3
    for _ in range(steps):
        R.step()
    R.sync()
    assert R.r.ctx.verify(R.stream) == -1
    plan = O.Plan(numel, W.CAP_BYTES, 2, n)
    rng = np.random.default_rng(rank)
    idx = rng.choice(plan.total, 1 << 14, replace=False)
    edges = np.concatenate([plan.bucket_off, plan.bucket_off + plan.bucket_padded - 1])
    idx = np.unique(np.concatenate([idx, edges])).astype(np.int64)
    bi = np.searchsorted(plan.bucket_off, idx, side="right") - 1
    used = ((idx - plan.bucket_off[bi]) < plan.bucket_used[bi]).astype(np.uint8)   # no 8 GB mask
    p, m, v, _ = O.run_sample(W.SEED, n, O.BF16, W.GRAD_SCALE, steps, idx, used, **HP_O)
    ti = torch.from_numpy(idx).to(R.r.p.device)
    np.testing.assert_array_equal(bits(R.r.p[ti].cpu().numpy()), bits(p), err_msg=f"p rank {rank}")
    # shard-local m, v: flat i in bucket b, shard r -> shard_off_b + (i - off_b - r E_b/n)
    b = np.searchsorted(plan.bucket_off, idx, side="right") - 1
    e = plan.bucket_padded[b] // n
    local = idx - plan.bucket_off[b] - rank * e
    mine = (local >= 0) & (local < e)
    j = (plan.bucket_off[b] // n + local)[mine]
    tj = torch.from_numpy(j).to(R.r.m.device)
    np.testing.assert_array_equal(bits(R.r.m[tj].cpu().numpy()), bits(m[mine]), err_msg=f"m rank {rank}")
    np.testing.assert_array_equal(bits(R.r.v[tj].cpu().numpy()), bits(v[mine]), err_msg=f"v rank {rank}")
    return R, int(mine.sum())


def model_parity(name):
    """SURVEY 8.d C2 model-mode parity at n > 1: GPT-2 small (stock PyTorch fwd/bwd, bf16
    autocast, random tokens per rank) through CheckmateDDP with per-bucket optimizer steps;
    every rank's pre-reduce gradients and pre-step state at sampled indices (+ bucket edges)
    go to rank 0, which recomputes the rank-order reduce and AdamW with the oracle and
    compares them with every rank's results bitwise; then the full checkpoint check."""
    from paper_2507_13522_b200.ddp import CheckmateDDP, GradProbe
    from paper_2507_13522_b200.modelbench import make_model
    from tests.model_parity import check_records, probe_indices
    n, rank = dist.get_world_size(), dist.get_rank()
    local = int(os.environ["LOCAL_RANK"])
    dev = torch.device("cuda", local)
    model = make_model(0).to(dev)
    model.train()
    cd = CheckmateDDP(model, local, n, rank, shm_name=name, ring_depth=9, persist_every=8)
    cd.probe = GradProbe(cd, probe_indices(cd, 1 << 14))
    g = torch.Generator(device=dev)
    g.manual_seed(1000 + rank)
    for _ in range(3):
        tok = torch.randint(0, 50257, (2, 256), device=dev, generator=g)
        cd.zero_grad()
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = model(tok, labels=tok).loss
        loss.backward()
        cd.step()
    torch.cuda.synchronize()
    st = cd.r.ctx.verify_ex(cm.CM_VERIFY_ALL, torch.cuda.current_stream())
    assert st == (cm.CM_OK, -1, None), st
    recs = [None] * n
    dist.all_gather_object(recs, cd.probe.records)
    if rank == 0:
        out = check_records(recs, n, W.HP)
        print(f"model parity: {out}", flush=True)
    return cd


def main():
    mode, name = sys.argv[1], sys.argv[2]
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = dist.get_world_size()
    if mode == "kd_rule":
        # R28: a host shadow across processes needs K >= 2 and D >= K + 1 (cm_connect)
        numel = W.numels(W.c1())
        try:
            harness.DistRank(numel, cm.CM_F32, 1 << 20, name + "a", 2, cm.CM_SHADOW_HOST, 0, persist_every=1)
            raise AssertionError("D=2, K=1 (-> 2) accepted")
        except cm.CMError as e:
            assert e.status == cm.CM_ERR_CONFIG, e
        R = harness.DistRank(numel, cm.CM_F32, 1 << 20, name, 3, cm.CM_SHADOW_HOST, 0, persist_every=1)
        assert R.r.ctx.info().persist_every == 2
        R.step()
        R.sync()
        rk = dist.get_rank()
        dist.barrier()
        R.r.ctx.finalize()
        for nm in (name, name + "a"):
            cm.unlink_shadow(nm, rk)
        dist.destroy_process_group()
        print(f"rank {rk}: {mode} ok", flush=True)
        return
    if mode == "model_parity":
        cd = model_parity(name)
        rk = dist.get_rank()
        dist.barrier()
        cd.finalize()
        cm.unlink_shadow(name, rk)
        dist.destroy_process_group()
        print(f"rank {rk}: {mode} ok", flush=True)
        return
    if mode == "llama_full_zero1":
        R, k = llama_full_zero1(name)
        dist.barrier()
        R.r.ctx.finalize()
        cm.unlink_shadow(name, R.rank_id)
        dist.destroy_process_group()
        print(f"rank {R.rank_id}: {mode} ok ({k} sampled shard elements)", flush=True)
        return
    dtype = cm.CM_BF16 if mode.endswith("bf16") else cm.CM_F32
    numel = W.numels(W.c1_ragged()) + [5, 70001]
    cap = 1 << 20
    plan = O.Plan(numel, cap, 4 if dtype == cm.CM_F32 else 2, n)
    opt = "sgd" if mode == "parity_sgd" else "adamw"
    hp_o = dict(lr=W.HP_SGD["lr"], momentum=W.HP_SGD["momentum"], wd=W.HP_SGD["weight_decay"]) \
        if opt == "sgd" else HP_O
    ref = O.Run(plan, seed=0, dtype=dtype, gscale=W.GRAD_SCALE, hp=hp_o, opt=opt)
    flags = cm.CM_FLAG_ATTACH if mode == "hardkill_phase2" else 0
    if mode.startswith("parity_zero1") or mode == "parity_bucket_step_zero1":
        flags |= cm.CM_FLAG_ZERO1
    if mode == "parity_oneshot_direct":
        flags |= cm.CM_FLAG_TAP_DIRECT
    if mode.startswith("parity_nvls"):
        flags |= cm.CM_FLAG_NVLS
    # host shadow across processes: persist_every K >= 2 and ring depth D >= K + 1 (cm.h)
    R = harness.DistRank(numel, dtype, cap, name, 3, cm.CM_SHADOW_HOST, flags, opt=opt, persist_every=2)
    if mode.startswith("parity_oneshot") or mode.startswith("parity_nvls") or mode == "parity_zero1_oneshot":
        # buckets up to 512 KiB / 1 MiB take the one-shot push kernel, the rest
        # the two-shot kernel; both must give the oracle's bits
        R.r.ctx.set_param("oneshot_max_bytes", (1 << 20) if "bf16" in mode else (512 << 10))
    if mode.startswith("parity_bucket_step"):
        # f1: each bucket's optimizer step right behind its all-reduce (cm_apply_bucket), in
        # reverse bucket order with the last two left to cm_apply_step
        c = R.r.ctx
        for t in range(6):
            c.gen_grads(R.seed, R.t, R.gscale, R.stream)
            for b in range(R.n_buckets):
                c.allreduce_multicast(b, R.t, R.stream)
            for b in reversed(range(2, R.n_buckets)):
                c.apply_bucket(b, R.t + 1, stream=R.stream, **R.hp)
            c.apply_step(R.t + 1, stream=R.stream, **R.hp)
            c.shadow_apply(R.t + 1, R.side)
            R.t += 1
            ref.step()
            R.sync()
            check(R, ref, f"iteration {t}", plan if mode.endswith("zero1") else None)
            st = c.verify_ex(cm.CM_VERIFY_ALL, R.stream)
            assert st == (cm.CM_OK, -1, None), st
    elif mode.startswith("parity"):
        for t in range(6):
            R.step()
            ref.step()
            R.sync()
            check(R, ref, f"iteration {t}", plan if mode.startswith("parity_zero1") else None)
            st = R.r.ctx.verify_ex(cm.CM_VERIFY_ALL, R.stream)
            assert st == (cm.CM_OK, -1, None), st
    elif mode == "nonfinite":
        # a NaN in rank n-1's gradients at an element of rank 0's shard, iteration 3: every
        # rank reports it (CM_ERR_INVARIANT, flat index), no shadow applies step 4, restore
        # returns 3 on every rank, and 3 more iterations match the oracle's clean run
        for _ in range(3):
            R.step()
            ref.step()
        R.sync()
        off, padded, used = R.r.ctx.bucket_info(0)
        i = off + min(used, padded // n) // 2
        c = R.r.ctx
        with torch.cuda.stream(R.stream):
            torch.cuda._sleep(int(120e6))          # every call is issued before the kernels run
        c.gen_grads(R.seed, R.t, R.gscale, R.stream)
        if R.rank_id == n - 1:
            with torch.cuda.stream(R.stream):
                R.r.grad[i] = float("nan")
        for b in range(R.n_buckets):
            c.allreduce_multicast(b, R.t, R.stream)
        c.apply_step(R.t + 1, stream=R.stream, **R.hp)
        c.shadow_apply(R.t + 1, R.side)
        R.t += 1
        R.sync()
        st = c.verify_ex(cm.CM_VERIFY_ALL, R.stream)
        assert st == (cm.CM_ERR_INVARIANT, i, "nonfinite"), st
        assert c.check() == (cm.CM_ERR_INVARIANT, 4, i)
        if R.rank_id == 0:
            assert c.info().shadow_step == 3
        torch.cuda.synchronize()
        dist.barrier()
        I = c.restore(R.stream)
        assert I == 3, I
        assert c.info().nonfinite_step == -1
        R.t = I
        for _ in range(3):
            R.step()
            ref.step()
        R.sync()
        check(R, ref, "after non-finite restore")
    elif mode == "restore_soft":
        for _ in range(4):
            R.step()
        R.sync()
        R.r.p.fill_(float("nan"))
        torch.cuda.synchronize()
        dist.barrier()
        I = R.r.ctx.restore(R.stream)
        assert I == 4, I
        for _ in range(4):
            ref.step()
        R.t = I
        for _ in range(3):
            R.step()
            ref.step()
        R.sync()
        check(R, ref, "after restore")
    elif mode == "hardkill_phase1":
        for _ in range(5):
            R.step()
        R.sync()
        dist.barrier()
        os._exit(0)        # die without finalize: the shadow segments stay in /dev/shm
    elif mode == "hardkill_phase2":
        # fresh process, garbage training state, attach to the surviving shadow segments
        R.r.p.fill_(float("nan"))
        R.r.m.fill_(float("nan"))
        torch.cuda.synchronize()
        dist.barrier()
        I = R.r.ctx.restore(R.stream)
        assert I == 5, I
        for _ in range(5):
            ref.step()
        R.t = I
        for _ in range(4):
            R.step()
            ref.step()
        R.sync()
        check(R, ref, "after hard-kill restore")
    dist.barrier()
    R.r.ctx.finalize()
    if mode != "hardkill_phase1":
        cm.unlink_shadow(name, R.rank_id)
    dist.destroy_process_group()
    print(f"rank {R.rank_id}: {mode} ok", flush=True)


if __name__ == "__main__":
    main()
