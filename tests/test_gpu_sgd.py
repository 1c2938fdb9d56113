"""GPU parity of the SGD-momentum optimizer (reading R27)
through the C ABI (cm_apply_step_sgd) against the CPU oracle, bit-exact: train state,
tap, shadow, ZeRO-1, restore roll-forward, and the full-size sampled GPT-2 case."""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2507_13522_b200 import cm, harness
from paper_2507_13522_b200 import workloads as W
from tests.gpu_util import bits, ring_flat, shadow_flat, t2np

pytestmark = pytest.mark.gpu

HP_O = dict(lr=W.HP_SGD["lr"], momentum=W.HP_SGD["momentum"], wd=W.HP_SGD["weight_decay"])
TABLES = {"ragged": W.numels(W.c1_ragged()), "mixed": [70000, 1, 3, 262145, 17, 5000, 300000, 2, 99999]}
_ctr = [0]


def _name():
    _ctr[0] += 1
    return f"cmsgd{os.getpid()}_{_ctr[0]}"


def make_group(numel, n, dtype=cm.CM_F32, D=2, flags=0, persist_every=1, hp=None):
    name = _name()
    g = harness.VirtualGroup(numel, n, 0, dtype, 1 << 20, name, D, cm.CM_SHADOW_HOST, flags, 0,
                             persist_every=persist_every, opt="sgd", hp=hp)
    g._shm = name
    return g


def close(g):
    g.sync()
    g.finalize()
    for r in range(g.n):
        cm.unlink_shadow(g._shm, r)


def oracle_for(numel, n, dtype, hp=None):
    plan = O.Plan(numel, 1 << 20, 4 if dtype == cm.CM_F32 else 2, n)
    h = dict(HP_O)
    if hp:
        h.update(hp)
    return plan, O.Run(plan, seed=0, dtype=dtype, gscale=W.GRAD_SCALE, hp=h, opt="sgd")


def _shard_of(flat, plan, rank):
    n = plan.world_size
    return np.concatenate([flat[o + rank * (p // n): o + (rank + 1) * (p // n)]
                           for o, p in zip(plan.bucket_off, plan.bucket_padded)])


@pytest.mark.parametrize("wd", [0.0, 1e-4])
@pytest.mark.parametrize("dtype", [cm.CM_F32, cm.CM_BF16])
@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_sgd_iterations_bit_exact(n, dtype, wd):
    numel = TABLES["ragged"]
    g = make_group(numel, n, dtype, hp=dict(weight_decay=wd))
    plan, ref = oracle_for(numel, n, dtype, hp=dict(wd=wd))
    try:
        for t in range(5):
            g.step()
            ref.step()
            g.sync()
            np.testing.assert_array_equal(bits(ring_flat(g, t % 2)), bits(ref.T), err_msg=f"tap t {t}")
            for r in g.ranks:
                np.testing.assert_array_equal(bits(t2np(r.grad)), bits(ref.R))
                np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p), err_msg=f"p rank {r.rank} t {t}")
                np.testing.assert_array_equal(bits(t2np(r.m)), bits(ref.m), err_msg=f"buf rank {r.rank} t {t}")
                assert not r.v.any()                                  # v untouched by SGD
                assert r.ctx.verify(g.stream) == -1
            sp, sm, sv = shadow_flat(g, (t + 1) & 1)
            np.testing.assert_array_equal(bits(sp), bits(ref.sp))
            np.testing.assert_array_equal(bits(sm), bits(ref.sm))
            assert not sv.any()
    finally:
        close(g)


@pytest.mark.parametrize("n", [2, 4])
def test_sgd_zero1_bit_exact(n):
    numel = TABLES["mixed"]
    g = make_group(numel, n, flags=cm.CM_FLAG_ZERO1)
    plan, ref = oracle_for(numel, n, cm.CM_F32)
    try:
        for t in range(4):
            g.step()
            ref.step()
            g.sync()
            for r in g.ranks:
                np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p), err_msg=f"p rank {r.rank} t {t}")
                np.testing.assert_array_equal(bits(t2np(r.m)), bits(_shard_of(ref.m, plan, r.rank)))
                assert r.ctx.verify(g.stream) == -1
    finally:
        close(g)


@pytest.mark.parametrize("K,D", [(1, 2), (4, 4)])
def test_sgd_restore_rolls_forward_bit_exact(K, D):
    """Kill at a step between host snapshots: restore replays the SGD records of the ring
    (optimizer kind + scalars per slot) and resumes identical to the uninterrupted run."""
    numel = TABLES["ragged"]
    n = 2
    kill_at = 2 * K + 1 if K > 1 else 5
    g = make_group(numel, n, D=D, persist_every=K)
    plan, ref = oracle_for(numel, n, cm.CM_F32)
    try:
        for _ in range(kill_at):
            g.step()
        g.sync()
        for r in g.ranks:
            r.p.fill_(float("nan")); r.m.fill_(float("nan"))
        torch.cuda.synchronize()
        assert [r.ctx.restore(g.stream) for r in g.ranks] == [kill_at] * n
        for _ in range(kill_at):
            ref.step()
        for r in g.ranks:
            np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p))
            np.testing.assert_array_equal(bits(t2np(r.m)), bits(ref.m))
            assert not r.v.any()
        g.t = kill_at
        for _ in range(3):
            g.step()
            ref.step()
        g.sync()
        for r in g.ranks:
            np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p))
            assert r.ctx.verify(g.stream) == -1
    finally:
        close(g)


def test_optimizer_switch_is_refused():
    g = make_group(TABLES["ragged"], 1)
    try:
        g.step()
        c = g.ranks[0].ctx
        c.gen_grads(0, 1, W.GRAD_SCALE, g.stream)
        for b in range(g.n_buckets):
            c.allreduce_multicast(b, 1, g.stream)
        with pytest.raises(cm.CMError) as e:
            c.apply_step(2, stream=g.stream)
        assert e.value.status == cm.CM_ERR_STATE
        c.apply_step_sgd(2, stream=g.stream, **W.HP_SGD)      # the context's own optimizer still works
    finally:
        close(g)


def test_sgd_gpt2_full_size_sampled():
    """GPT-2 small at full size (17 buckets), n=2 virtual ranks, 3 SGD steps: sampled
    elements (incl. every bucket edge) vs the oracle's per-element trajectories."""
    numel = W.numels(W.gpt2_small())
    n = 2
    name = _name()
    g = harness.VirtualGroup(numel, n, 0, cm.CM_F32, W.CAP_BYTES, name, 2, cm.CM_SHADOW_HOST, 0, 0, opt="sgd")
    g._shm = name
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
        p, b, R = O.run_sample_sgd(0, n, O.F32, W.GRAD_SCALE, steps, idx, used, **HP_O)
        for r in g.ranks:
            ti = torch.from_numpy(idx).to(r.p.device)
            np.testing.assert_array_equal(bits(r.p[ti].cpu().numpy()), bits(p))
            np.testing.assert_array_equal(bits(r.m[ti].cpu().numpy()), bits(b))
            np.testing.assert_array_equal(bits(r.grad[ti].cpu().numpy()), bits(R))
            assert r.ctx.verify(g.stream) == -1
    finally:
        close(g)
