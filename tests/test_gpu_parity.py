"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by
element, bit-exact (north_star: "The GPU path must match the oracle bit-exactly").

Ranks are virtual ranks on one GPU (n contexts in one process, issued on one stream): the
kernels and data path are the ones the multi-GPU run uses; only the cross-GPU flag barrier
is off (B200_PROFILING.md forbids kernels that wait on each other on one GPU).
"""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2507_13522_b200 import cm, harness
from paper_2507_13522_b200 import workloads as W
from tests.gpu_util import assemble, bits, host_array, ring_flat, shadow_flat, t2np

pytestmark = pytest.mark.gpu

HP_O = dict(lr=W.HP["lr"], b1=W.HP["beta1"], b2=W.HP["beta2"], eps=W.HP["eps"], wd=W.HP["weight_decay"])
_name_ctr = [0]


def _name():
    _name_ctr[0] += 1
    return f"cmt{os.getpid()}_{_name_ctr[0]}"


def make_group(numel, n, dtype=cm.CM_F32, cap=1 << 20, D=2, place=cm.CM_SHADOW_HOST, flags=0, seed=0):
    name = _name()
    g = harness.VirtualGroup(numel, n, 0, dtype, cap, name, D, place, flags, seed)
    g._shm = name
    return g


def close(g):
    g.sync()
    g.finalize()
    for r in range(g.n):
        cm.unlink_shadow(g._shm, r)


def oracle_for(numel, n, dtype, cap, seed=0):
    plan = O.Plan(numel, cap, 4 if dtype == cm.CM_F32 else 2, n)
    return plan, O.Run(plan, seed=seed, dtype=dtype, gscale=W.GRAD_SCALE, hp=HP_O)


TABLES = {"c1": W.numels(W.c1()), "ragged": W.numels(W.c1_ragged()),
          "mixed": [70000, 1, 3, 262145, 17, 5000, 300000, 2, 99999]}


@pytest.mark.parametrize("dtype", [cm.CM_F32, cm.CM_BF16])
@pytest.mark.parametrize("n", [1, 2, 3, 8])
def test_inputs_match_oracle_generator(dtype, n):
    numel = TABLES["ragged"]
    g = make_group(numel, n, dtype)
    plan = O.Plan(numel, 1 << 20, 4 if dtype == 0 else 2, n)
    try:
        g.gen(t=7)
        g.sync()
        for r in g.ranks:
            np.testing.assert_array_equal(t2np(r.grad), O.gen_grads(plan, 0, r.rank, 7, dtype, W.GRAD_SCALE))
            np.testing.assert_array_equal(bits(t2np(r.p)), bits(O.gen_p0(plan, 0)))
            assert not r.m.any() and not r.v.any()
    finally:
        close(g)


@pytest.mark.parametrize("table", ["c1", "ragged", "mixed"])
@pytest.mark.parametrize("dtype", [cm.CM_F32, cm.CM_BF16])
@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_iterations_bit_exact(table, dtype, n):
    """Every element of R, the tap ring, train p/m/v and shadow p/m/v, every iteration."""
    numel = TABLES[table]
    iters = 10 if table == "c1" else 4
    g = make_group(numel, n, dtype)
    plan, ref = oracle_for(numel, n, dtype, 1 << 20)
    try:
        for t in range(iters):
            g.step()
            ref.step()
            g.sync()
            for r in g.ranks:
                np.testing.assert_array_equal(bits(t2np(r.grad)), bits(ref.R), err_msg=f"R rank {r.rank} t {t}")
            np.testing.assert_array_equal(bits(ring_flat(g, t % 2)), bits(ref.T), err_msg=f"tap t {t}")
            for r in g.ranks:
                for name, a, b in (("p", r.p, ref.p), ("m", r.m, ref.m), ("v", r.v, ref.v)):
                    np.testing.assert_array_equal(bits(t2np(a)), bits(b), err_msg=f"{name} rank {r.rank} t {t}")
            sp, sm, sv = shadow_flat(g, (t + 1) & 1)
            for name, a, b in (("sp", sp, ref.sp), ("sm", sm, ref.sm), ("sv", sv, ref.sv)):
                np.testing.assert_array_equal(bits(a), bits(b), err_msg=f"shadow {name} t {t}")
            for r in g.ranks:
                assert r.ctx.verify(g.stream) == -1
                assert r.ctx.info().shadow_step == t + 1
    finally:
        close(g)


@pytest.mark.parametrize("n", [2, 4, 8])
def test_reduce_within_1e6_of_fp64(n):
    numel = TABLES["c1"]
    g = make_group(numel, n)
    plan = O.Plan(numel, 1 << 20, 4, n)
    try:
        g.gen(t=0)
        g.allreduce(t=0)
        g.sync()
        R = t2np(g.ranks[0].grad).astype(np.float64)
        G = np.stack([O.gen_grads(plan, 0, r, 0, O.F32) for r in range(n)]).astype(np.float64)
        err = np.abs(R - G.sum(0))
        assert np.all(err <= 1e-6 * np.abs(G).sum(0))
    finally:
        close(g)


def test_device_shadow_placement_bit_exact():
    numel = TABLES["ragged"]
    g = make_group(numel, 2, place=cm.CM_SHADOW_DEVICE)
    plan, ref = oracle_for(numel, 2, cm.CM_F32, 1 << 20)
    try:
        for t in range(5):
            g.step()
            ref.step()
            g.sync()
            for r in g.ranks:
                assert r.ctx.verify(g.stream) == -1
            np.testing.assert_array_equal(bits(t2np(g.ranks[1].p)), bits(ref.p))
    finally:
        close(g)


@pytest.mark.parametrize("n", [1, 4])
@pytest.mark.parametrize("flag", [cm.CM_FLAG_TAP_COPYENGINE, cm.CM_FLAG_TAP_DIRECT])
def test_copy_engine_tap_modes_bit_exact(flag, n):
    numel = TABLES["ragged"]
    g = make_group(numel, n, flags=flag)
    plan, ref = oracle_for(numel, n, cm.CM_F32, 1 << 20)
    try:
        for t in range(5):
            g.step()
            ref.step()
            g.sync()
            np.testing.assert_array_equal(bits(ring_flat(g, t % 2)), bits(ref.T))
            for r in g.ranks:
                assert r.ctx.verify(g.stream) == -1
    finally:
        close(g)


def test_no_tap_mode_matches_train_state():
    numel = TABLES["c1"]
    g = make_group(numel, 2, flags=cm.CM_FLAG_NO_TAP)
    plan, ref = oracle_for(numel, 2, cm.CM_F32, 1 << 20)
    try:
        for t in range(3):
            g.step()
            ref.step()
        g.sync()
        np.testing.assert_array_equal(bits(t2np(g.ranks[0].p)), bits(ref.p))
        with pytest.raises(cm.CMError):
            g.ranks[0].ctx.shadow_apply(4, g.side)
    finally:
        close(g)


def test_tap_exactly_once_covers_every_element():
    """Poison the ring; after one iteration every element of every rank's slot was written
    once with R (sum over ranks of tapped elements = padded elements, S)."""
    numel = TABLES["ragged"]
    n = 4
    g = make_group(numel, n)
    plan, ref = oracle_for(numel, n, cm.CM_F32, 1 << 20)
    try:
        info = g.ranks[0].ctx.info()
        for r in g.ranks:
            ptr = r.ctx.ring_view(0)
            import ctypes as C
            C.memset(ptr, 0x7F, info.shard_numel * 4)   # 0x7F7F7F7F: finite poison never produced
        g.step()
        ref.step()
        g.sync()
        flat = ring_flat(g, 0)
        assert not np.any(flat.view(np.uint32) == 0x7F7F7F7F)
        np.testing.assert_array_equal(flat.view(np.uint32), ref.T.view(np.uint32))
        assert n * info.shard_numel == plan.total
    finally:
        close(g)


def test_flow_control_refuses_to_overwrite_unconsumed_slot():
    numel = TABLES["c1"]
    g = make_group(numel, 2, D=2)
    try:
        g.step(shadow=False)          # iteration 0 -> slot 0, not consumed
        g.step(shadow=False)          # iteration 1 -> slot 1
        g.gen()
        with pytest.raises(cm.CMError) as e:
            g.allreduce()             # iteration 2 would overwrite slot 0
        assert e.value.status == cm.CM_ERR_STATE
        g.shadow(step=1)              # slot 0 released: the same call now succeeds
        g.allreduce()
        g.apply()
        g.t += 1
        g.shadow(step=2)
        g.shadow(step=3)
        g.sync()
        for r in g.ranks:
            assert r.ctx.verify(g.stream) == -1
    finally:
        close(g)


def test_backpressure_with_slow_shadow_is_lossless():
    """The shadow stream is throttled (sleep kernels): training blocks on the ring, never
    overwrites, and the shadow stays bit-identical."""
    numel = TABLES["ragged"]
    g = make_group(numel, 2, D=2)
    plan, ref = oracle_for(numel, 2, cm.CM_F32, 1 << 20)
    try:
        for t in range(8):
            with torch.cuda.stream(g.side):
                torch.cuda._sleep(20_000_000)      # ~10 ms at 2 GHz before each shadow step
            g.step()
            ref.step()
        g.sync()
        np.testing.assert_array_equal(bits(t2np(g.ranks[0].p)), bits(ref.p))
        sp, sm, sv = shadow_flat(g, 8 & 1)
        np.testing.assert_array_equal(bits(sp), bits(ref.sp))
        np.testing.assert_array_equal(bits(sv), bits(ref.sv))
    finally:
        close(g)


def test_state_errors():
    numel = TABLES["c1"]
    g = make_group(numel, 2)
    try:
        c = g.ranks[0].ctx
        with pytest.raises(cm.CMError) as e:
            c.apply_step(1, stream=g.stream)            # before any all-reduce
        assert e.value.status == cm.CM_ERR_STATE
        with pytest.raises(cm.CMError) as e:
            c.allreduce_multicast(0, 5, g.stream)       # iteration gap
        assert e.value.status == cm.CM_ERR_STATE
        with pytest.raises(cm.CMError) as e:
            c.allreduce_multicast(99, 0, g.stream)      # bucket out of range
        assert e.value.status == cm.CM_ERR_ARG
        c.allreduce_multicast(0, 0, g.stream)
        with pytest.raises(cm.CMError) as e:
            c.allreduce_multicast(0, 0, g.stream)       # same bucket twice
        assert e.value.status == cm.CM_ERR_STATE
        with pytest.raises(cm.CMError) as e:
            c.apply_step(1, stream=g.stream)            # partial iteration: no partial update
        assert e.value.status == cm.CM_ERR_STATE
        with pytest.raises(cm.CMError) as e:
            c.shadow_apply(1, g.side)                   # before cm_apply_step(1)
        assert e.value.status == cm.CM_ERR_STATE
    finally:
        close(g)


@pytest.mark.parametrize("lag", [0, 1])
@pytest.mark.parametrize("n", [2, 4])
def test_soft_restore_continues_bit_exact(n, lag):
    """Kill (poison the training state) at iteration k, restore from the shadow, continue:
    identical to the uninterrupted run (PAPER.md:601 methodology)."""
    numel = TABLES["ragged"]
    k, more = 5, 5
    g = make_group(numel, n, D=2)
    plan, ref = oracle_for(numel, n, cm.CM_F32, 1 << 20)
    try:
        for t in range(k):
            g.step(shadow=(t < k - lag))              # lag=1: the shadow misses the last step
        g.sync()
        for r in g.ranks:
            r.p.fill_(float("nan")); r.m.fill_(float("nan")); r.v.fill_(float("nan"))
        torch.cuda.synchronize()
        steps = [r.ctx.restore(g.stream) for r in g.ranks]
        assert steps == [k] * n                       # roll-forward recovers the lagging step
        for _ in range(k):
            ref.step()
        for r in g.ranks:
            np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p))
            np.testing.assert_array_equal(bits(t2np(r.m)), bits(ref.m))
            np.testing.assert_array_equal(bits(t2np(r.v)), bits(ref.v))
        g.t = k
        for _ in range(more):
            g.step()
            ref.step()
        g.sync()
        for r in g.ranks:
            np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p))
            assert r.ctx.verify(g.stream) == -1
    finally:
        close(g)


@pytest.mark.parametrize("n", [1, 8])
def test_gpt2_full_size_sampled(n):
    """GPT-2 small at full size (124,439,808 params, 17 buckets): 3 iterations, sampled
    elements vs the oracle's per-element trajectories (PAPER.md:306-308 independence)."""
    numel = W.numels(W.gpt2_small())
    g = make_group(numel, n, cap=W.CAP_BYTES)
    try:
        steps = 3
        for _ in range(steps):
            g.step()
        g.sync()
        plan = O.Plan(numel, W.CAP_BYTES, 4, n)
        rng = np.random.default_rng(0)
        idx = rng.choice(plan.total, 1 << 15, replace=False)
        edges = np.concatenate([plan.bucket_off, plan.bucket_off + plan.bucket_padded - 1])
        idx = np.unique(np.concatenate([idx, edges])).astype(np.int64)
        used = plan.used_mask()[idx]
        p, m, v, R = O.run_sample(0, n, O.F32, W.GRAD_SCALE, steps, idx, used, **HP_O)
        for r in g.ranks:
            ti = torch.from_numpy(idx).to(r.p.device)
            np.testing.assert_array_equal(bits(r.p[ti].cpu().numpy()), bits(p))
            np.testing.assert_array_equal(bits(r.m[ti].cpu().numpy()), bits(m))
            np.testing.assert_array_equal(bits(r.v[ti].cpu().numpy()), bits(v))
            np.testing.assert_array_equal(bits(r.grad[ti].cpu().numpy()), bits(R))
            assert r.ctx.verify(g.stream) == -1
    finally:
        close(g)


def test_llama_shaped_bf16_sampled():
    """Llama-3-8B-shaped layers (first 2 decoder layers + norms, bf16 grads, 25 MiB cap,
    dedicated buckets for the big matrices) at n=8, sampled vs the oracle."""
    t = W.llama3_8b()
    numel = [x for _, x in t[1:19]] + [4096]       # 2 layers + final norm (no 1 GB embeddings)
    n = 8
    g = make_group(numel, n, dtype=cm.CM_BF16, cap=W.CAP_BYTES)
    try:
        for _ in range(2):
            g.step()
        g.sync()
        plan = O.Plan(numel, W.CAP_BYTES, 2, n)
        idx = np.unique(np.random.default_rng(1).choice(plan.total, 1 << 15, replace=False)).astype(np.int64)
        used = plan.used_mask()[idx]
        p, m, v, R = O.run_sample(0, n, O.BF16, W.GRAD_SCALE, 2, idx, used, **HP_O)
        r = g.ranks[3]
        ti = torch.from_numpy(idx).to(r.p.device)
        np.testing.assert_array_equal(bits(r.p[ti].cpu().numpy()), bits(p))
        np.testing.assert_array_equal(bits(r.v[ti].cpu().numpy()), bits(v))
        Rg = (t2np(r.grad[ti]).astype(np.uint32) << 16).view(np.float32)
        np.testing.assert_array_equal(bits(Rg), bits(R))
        for rr in g.ranks:
            assert rr.ctx.verify(g.stream) == -1
    finally:
        close(g)


@pytest.mark.parametrize("impl", [0, 1, 2, 3])
@pytest.mark.parametrize("dtype", [cm.CM_F32, cm.CM_BF16])
def test_adamw_implementations_bit_exact(impl, dtype):
    """Every AdamW data-movement variant (vectorised, TMA-staged, warp-tiled pair, warp-tiled
    single tile) computes the
    same bits: the arithmetic is one device function; only the loads/stores differ."""
    numel = TABLES["mixed"]
    g = make_group(numel, 2, dtype)
    for r in g.ranks:
        r.ctx.set_param("adamw_impl", impl)
    plan, ref = oracle_for(numel, 2, dtype, 1 << 20)
    try:
        for t in range(3):
            g.step()
            ref.step()
        g.sync()
        for r in g.ranks:
            np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p))
            np.testing.assert_array_equal(bits(t2np(r.m)), bits(ref.m))
            np.testing.assert_array_equal(bits(t2np(r.v)), bits(ref.v))
            assert r.ctx.verify(g.stream) == -1
    finally:
        close(g)


@pytest.mark.parametrize("blocks", [1, 7, 148, 1024])
def test_grid_invariance(blocks):
    """Element-local math: any grid gives identical bytes (SURVEY 8.c grid invariance)."""
    numel = TABLES["ragged"]
    g = make_group(numel, 1)
    for r in g.ranks:
        r.ctx.set_param("ar_blocks_tap_only", blocks)
        r.ctx.set_param("ar_blocks", blocks)
        r.ctx.set_param("adam_blocks", blocks)
        r.ctx.set_param("shadow_blocks", blocks)
    plan, ref = oracle_for(numel, 1, cm.CM_F32, 1 << 20)
    try:
        for t in range(2):
            g.step()
            ref.step()
        g.sync()
        np.testing.assert_array_equal(bits(t2np(g.ranks[0].p)), bits(ref.p))
        np.testing.assert_array_equal(bits(ring_flat(g, 1)), bits(ref.T))
        assert g.ranks[0].ctx.verify(g.stream) == -1
    finally:
        close(g)


@pytest.mark.parametrize("K,D", [(2, 2), (4, 4), (4, 6)])
def test_persist_every_k_restore_rolls_forward(K, D):
    """Host snapshot every K steps; the ring logs the steps between.  After a failure at any
    step, restore rolls forward from the last snapshot over the ring and resumes bit-exact."""
    numel = TABLES["ragged"]
    n = 2
    for kill_at in (K + 1, 2 * K, 2 * K + 1):
        name = _name()
        g = harness.VirtualGroup(numel, n, 0, cm.CM_F32, 1 << 20, name, D, cm.CM_SHADOW_HOST, 0, 0,
                                 persist_every=K)
        g._shm = name
        plan, ref = oracle_for(numel, n, cm.CM_F32, 1 << 20)
        try:
            for t in range(kill_at):
                g.step()
            g.sync()
            for r in g.ranks:
                assert r.ctx.verify(g.stream) == -1
                r.p.fill_(float("nan")); r.m.fill_(float("nan")); r.v.fill_(float("nan"))
            torch.cuda.synchronize()
            steps = [r.ctx.restore(g.stream) for r in g.ranks]
            assert steps == [kill_at] * n, (steps, kill_at)
            for _ in range(kill_at):
                ref.step()
            for r in g.ranks:
                np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p))
                np.testing.assert_array_equal(bits(t2np(r.v)), bits(ref.v))
            g.t = kill_at
            for _ in range(2 * K + 1):
                g.step()
                ref.step()
            g.sync()
            for r in g.ranks:
                np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p))
                assert r.ctx.verify(g.stream) == -1
        finally:
            close(g)


def test_consolidation_min_rule_across_lagging_shards():
    """Shards at different shadow steps (rank 1's shadow stops 2 steps early, its ring still
    holds the taps): I = min over shards of the reachable step; both end bit-exact at I."""
    numel = TABLES["ragged"]
    n = 2
    g = make_group(numel, n, D=4)
    plan, ref = oracle_for(numel, n, cm.CM_F32, 1 << 20)
    try:
        for t in range(6):
            g.gen()
            g.allreduce()
            g.apply()
            g.ranks[0].ctx.shadow_apply(t + 1, g.side)
            if t < 4:
                g.ranks[1].ctx.shadow_apply(t + 1, g.side)
            g.t += 1
        g.sync()
        assert [r.ctx.info().shadow_step for r in g.ranks] == [6, 4]
        steps = [r.ctx.restore(g.stream) for r in g.ranks]
        assert steps == [6, 6]                      # rank 1 rolls forward over its ring
        for _ in range(6):
            ref.step()
        for r in g.ranks:
            np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p))
            assert r.ctx.verify(g.stream) == -1
    finally:
        close(g)


def test_lagging_shadow_falls_back_from_staging_to_ring():
    """The shadow normally reads the reduced shard from the tap's HBM staging half; when it
    lags so far that the half was reused, it reads the host ring instead.  Both bit-exact."""
    numel = TABLES["ragged"]
    n = 2
    g = make_group(numel, n, D=4)
    plan, ref = oracle_for(numel, n, cm.CM_F32, 1 << 20)
    try:
        for _ in range(3):
            g.step(shadow=False)        # iterations 0,1,2: staging half 0 now holds iteration 2
            ref.step()
        g.shadow(step=1)                # iteration 0: staging reused -> host ring
        g.shadow(step=2)                # iteration 1: staging half 1
        g.shadow(step=3)                # iteration 2: staging half 0
        g.sync()
        for r in g.ranks:
            assert r.ctx.verify(g.stream) == -1
        sp, sm, sv = shadow_flat(g, 3 & 1)
        np.testing.assert_array_equal(bits(sp), bits(ref.sp))
        np.testing.assert_array_equal(bits(sv), bits(ref.sv))
    finally:
        close(g)


def _zero1_shard_of(flat, plan, rank):
    """The oracle's flat array restricted to `rank`'s shard, in shard-local order."""
    n = plan.world_size
    out = []
    for off, padded in zip(plan.bucket_off, plan.bucket_padded):
        e = padded // n
        out.append(flat[off + rank * e: off + (rank + 1) * e])
    return np.concatenate(out)


@pytest.mark.parametrize("zimpl", [1, 0, 2])
@pytest.mark.parametrize("dtype", [cm.CM_F32, cm.CM_BF16])
@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_zero1_bit_exact(n, dtype, zimpl):
    """ZeRO-1 (f3): reduce-scatter + tap, AdamW on the own shard, fused parameter
    all-gather.  Every rank's full p, its shard-local m/v and the shadow equal the oracle
    (the unsharded definition) bit for bit, with two groups per thread in flight (default),
    with one, and with the parameter all-gather pushed by bulk copies (zero1_impl 2)."""
    numel = TABLES["mixed"]
    g = make_group(numel, n, dtype, flags=cm.CM_FLAG_ZERO1)
    for r in g.ranks:
        r.ctx.set_param("zero1_impl", zimpl)
    plan, ref = oracle_for(numel, n, dtype, 1 << 20)
    try:
        assert g.ranks[0].m.numel() == plan.total // n
        for t in range(4):
            g.step()
            ref.step()
            g.sync()
            for r in g.ranks:
                np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p), err_msg=f"p rank {r.rank} t {t}")
                np.testing.assert_array_equal(bits(t2np(r.m)), bits(_zero1_shard_of(ref.m, plan, r.rank)))
                np.testing.assert_array_equal(bits(t2np(r.v)), bits(_zero1_shard_of(ref.v, plan, r.rank)))
                assert r.ctx.verify(g.stream) == -1
            np.testing.assert_array_equal(bits(ring_flat(g, t % 2)), bits(ref.T), err_msg=f"tap t {t}")
    finally:
        close(g)


def test_zero1_restore_bit_exact():
    numel = TABLES["ragged"]
    n = 4
    g = make_group(numel, n, flags=cm.CM_FLAG_ZERO1, D=4)
    plan, ref = oracle_for(numel, n, cm.CM_F32, 1 << 20)
    try:
        for _ in range(5):
            g.step()
        g.sync()
        for r in g.ranks:
            r.p.fill_(float("nan")); r.m.fill_(float("nan")); r.v.fill_(float("nan"))
        torch.cuda.synchronize()
        assert [r.ctx.restore(g.stream) for r in g.ranks] == [5] * n
        for _ in range(5):
            ref.step()
        g.t = 5
        for _ in range(3):
            g.step()
            ref.step()
        g.sync()
        for r in g.ranks:
            np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p))
            np.testing.assert_array_equal(bits(t2np(r.v)), bits(_zero1_shard_of(ref.v, plan, r.rank)))
            assert r.ctx.verify(g.stream) == -1
    finally:
        close(g)


def test_checkpoint_file_save_load_restore(tmp_path):
    """f4: persist every rank's host shadow to a CheckpointFile (CRC-32), drop the shared
    memory, recreate it from the files (as on a new host), attach, restore, continue:
    bit-exact vs the oracle."""
    numel = TABLES["ragged"]
    n = 2
    g = make_group(numel, n, D=4)
    g.ranks[0].ctx  # noqa: B018
    plan, ref = oracle_for(numel, n, cm.CM_F32, 1 << 20)
    try:
        for _ in range(5):
            g.step()
        g.sync()
        for r in g.ranks:
            r.ctx.join(g.stream)
        g.stream.synchronize()
        for r in range(n):
            cm.shadow_save(g._shm, r, tmp_path / f"rank{r}.ckpt")
    finally:
        close(g)                                   # segments unlinked: only the files remain
    name = _name()
    for r in range(n):
        cm.shadow_load(tmp_path / f"rank{r}.ckpt", name, r)
    g2 = harness.VirtualGroup(numel, n, 0, cm.CM_F32, 1 << 20, name, 4, cm.CM_SHADOW_HOST, cm.CM_FLAG_ATTACH, 0)
    g2._shm = name
    try:
        for r in g2.ranks:
            r.p.fill_(float("nan"))
        torch.cuda.synchronize()
        assert [r.ctx.restore(g2.stream) for r in g2.ranks] == [5] * n
        for _ in range(5):
            ref.step()
        g2.t = 5
        for _ in range(3):
            g2.step()
            ref.step()
        g2.sync()
        for r in g2.ranks:
            np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p))
            assert r.ctx.verify(g2.stream) == -1
    finally:
        close(g2)


@pytest.mark.parametrize("drain", [0, 1, 2])
def test_drain_modes_ring_and_restore_bit_exact(drain):
    """The tap drain and the snapshot persist by copy engine (0) or by the SM drain kernel
    (1, 2 CTAs): the ring holds T exactly, the host snapshot equals the shadow, and a restore
    that rolls forward over the ring resumes bit-exact."""
    numel = TABLES["ragged"]
    n, K, D = 2, 4, 4
    name = _name()
    g = harness.VirtualGroup(numel, n, 0, cm.CM_F32, 1 << 20, name, D, cm.CM_SHADOW_HOST, 0, 0, persist_every=K)
    g._shm = name
    for r in g.ranks:
        r.ctx.set_param("drain_ctas", drain)
    plan, ref = oracle_for(numel, n, cm.CM_F32, 1 << 20)
    try:
        kill_at = 2 * K + 1
        for t in range(kill_at):
            g.step()
            ref.step()
            g.sync()
            for r in g.ranks:
                r.ctx.join(g.stream)
            g.stream.synchronize()
            np.testing.assert_array_equal(bits(ring_flat(g, t % D)), bits(ref.T), err_msg=f"ring t {t}")
            assert all(r.ctx.info().drain_ctas == drain for r in g.ranks)
        for r in g.ranks:
            assert r.ctx.verify(g.stream) == -1
            r.p.fill_(float("nan")); r.m.fill_(float("nan")); r.v.fill_(float("nan"))
        torch.cuda.synchronize()
        assert [r.ctx.restore(g.stream) for r in g.ranks] == [kill_at] * n
        for r in g.ranks:
            np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p))
            np.testing.assert_array_equal(bits(t2np(r.v)), bits(ref.v))
    finally:
        close(g)


@pytest.mark.parametrize("impl", [1, 2])
@pytest.mark.parametrize("dtype", [cm.CM_F32, cm.CM_BF16])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_pipelined_allreduce_kernel_bit_exact(n, dtype, impl):
    """ar_impl=1 (software-pipelined two-shot kernel, one block per SM) and ar_impl=2 (bulk-copy
    pipeline: TMA pulls of every rank's tile into shared memory, bulk-store pushes of the
    result; ragged last tiles): same bits."""
    if impl == 2 and n == 1:
        pytest.skip("ar_impl 2 is the multi-rank kernel (n = 1 has no reduction)")
    numel = TABLES["mixed"] + [3 * 4096 + 8, 12288 * 3 // 4 + 16]
    g = make_group(numel, n, dtype)
    for r in g.ranks:
        r.ctx.set_param("ar_impl", impl)
        r.ctx.set_param("ar_pipe_blocks", 7)      # several vectors per thread on these sizes
    plan, ref = oracle_for(numel, n, dtype, 1 << 20)
    try:
        for t in range(3):
            g.step()
            ref.step()
            g.sync()
            for r in g.ranks:
                np.testing.assert_array_equal(bits(t2np(r.grad)), bits(ref.R), err_msg=f"R rank {r.rank} t {t}")
                np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p))
                assert r.ctx.verify(g.stream) == -1
            np.testing.assert_array_equal(bits(ring_flat(g, t % 2)), bits(ref.T), err_msg=f"tap t {t}")
    finally:
        close(g)


@pytest.mark.parametrize("impl", [2, 0, 1])
@pytest.mark.parametrize("dtype", [cm.CM_F32, cm.CM_BF16])
def test_adamw_zero_gradients_bit_exact(dtype, impl):
    """Exact zeros through the AdamW divisions (the zero-operand fast path of div_rn_z /
    sqrt_rn_z): elements whose gradient is +0 or -0 on every rank at every step (moments stay
    0: 0/bc1, 0/bc2, sqrt(0), 0/eps), elements zero only at some steps, and the rest
    generated.  Train, shadow and tap equal the oracle bit for bit."""
    import torch
    numel = TABLES["mixed"]
    n = 2
    g = make_group(numel, n, dtype)
    for r in g.ranks:
        r.ctx.set_param("adamw_impl", impl)
    plan, ref = oracle_for(numel, n, dtype, 1 << 20)
    idx = np.arange(plan.total)
    always = idx % 3 == 0
    neg = (idx % 6 == 3) & plan.used_mask()
    try:
        for t in range(4):
            grads = [O.gen_grads(plan, 0, r, t, dtype, W.GRAD_SCALE).copy() for r in range(n)]
            sometimes = (idx + t) % 5 == 0
            for a in grads:
                a[always | sometimes] = 0
                a[neg & ~always] = 0x8000 if dtype == cm.CM_BF16 else np.float32(-0.0)
            for r, a in zip(g.ranks, grads):
                src = torch.from_numpy(a.view(np.int16) if dtype == cm.CM_BF16 else a)
                if dtype == cm.CM_BF16:
                    r.grad.view(torch.int16).copy_(src)
                else:
                    r.grad.copy_(src)
            torch.cuda.synchronize()
            g.step(gen=False)
            ref.step(grads=grads)
            g.sync()
            for r in g.ranks:
                np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p), err_msg=f"p t {t}")
                np.testing.assert_array_equal(bits(t2np(r.m)), bits(ref.m), err_msg=f"m t {t}")
                np.testing.assert_array_equal(bits(t2np(r.v)), bits(ref.v), err_msg=f"v t {t}")
                assert r.ctx.verify(g.stream) == -1
            np.testing.assert_array_equal(bits(ring_flat(g, t % 2)), bits(ref.T), err_msg=f"tap t {t}")
        assert np.count_nonzero(bits(t2np(g.ranks[0].m))[always] != 0) == 0
    finally:
        close(g)


def test_restore_keeps_its_source_snapshot_when_a_shard_ran_ahead():
    """A shard whose shadow ran past the consolidation point I (rank 0 persisted step 8,
    rank 1 can only reach 6): restore rolls rank 0 forward from its step-4 snapshot and
    persists step 6 into the half holding the stale step 8 -- never over the step-4 source,
    so a kill during that persist still leaves a half from which I is reachable.  Both
    shards end bit-exact at I and continue bit-exact."""
    from tests.gpu_util import shard_slices
    numel = TABLES["ragged"]
    n, K, D = 2, 4, 8
    name = _name()
    g = harness.VirtualGroup(numel, n, 0, cm.CM_F32, 1 << 20, name, D, cm.CM_SHADOW_HOST, 0, 0,
                             persist_every=K)
    g._shm = name
    plan, ref = oracle_for(numel, n, cm.CM_F32, 1 << 20)
    r0, r1 = g.ranks
    try:
        for _ in range(4):                                   # both shards persist step 4
            g.step()
        for t in (4, 5):                                     # both train; only rank 0's shadow
            g.gen(t)
            g.allreduce(t)
            g.apply(t + 1)
            r0.ctx.shadow_apply(t + 1, g.side)
        for t in (6, 7):                                     # rank 0 alone runs ahead to step 8
            r0.ctx.gen_grads(g.seed, t, g.gscale, g.stream)
            for b in range(g.n_buckets):
                r0.ctx.allreduce_multicast(b, t, g.stream)
            r0.ctx.apply_step(t + 1, stream=g.stream, **g.hp)
            r0.ctx.shadow_apply(t + 1, g.side)
        g.sync()
        assert [r.ctx.info().shadow_step for r in g.ranks] == [8, 4]
        for r in g.ranks:
            r.p.fill_(float("nan")); r.m.fill_(float("nan")); r.v.fill_(float("nan"))
        torch.cuda.synchronize()
        steps = [r.ctx.restore(g.stream) for r in g.ranks]
        g.sync()
        assert steps == [6, 6], steps
        for _ in range(4):
            ref.step()
        p4 = ref.p.copy()
        for _ in range(2):
            ref.step()
        for r in g.ranks:
            np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p))
            np.testing.assert_array_equal(bits(t2np(r.m)), bits(ref.m))
            np.testing.assert_array_equal(bits(t2np(r.v)), bits(ref.v))
        # rank 0's step-4 snapshot (the restore's source) survived the step-6 persist
        L = r0.ctx.info().shard_numel
        want = np.zeros(L, np.float32)
        for lo, hi, s in shard_slices(r0):
            want[s:s + (hi - lo)] = p4[lo:hi]
        halves = [host_array(r0.ctx.shadow_view(h)[0], L, np.float32) for h in (0, 1)]
        assert any(np.array_equal(bits(hp), bits(want)) for hp in halves)
        g.t = 6
        for _ in range(3):
            g.step()
            ref.step()
        g.sync()
        for r in g.ranks:
            np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p))
            assert r.ctx.verify(g.stream) == -1
    finally:
        close(g)
