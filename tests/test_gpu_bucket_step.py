"""Per-bucket optimizer steps (cm_apply_bucket): the optimizer
of each bucket runs right behind its all-reduce, and cm_apply_step finishes the step.  Every
element of R, train p/m/v, the tap ring and the shadow equals the oracle's whole-buffer step,
bitwise, for AdamW and SGD, replicated and ZeRO-1, fp32 and bf16 gradients, virtual ranks."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2507_13522_b200 import cm, harness
from paper_2507_13522_b200 import workloads as W
from tests.gpu_util import bits, ring_flat, shadow_flat, t2np

pytestmark = pytest.mark.gpu

NUMEL = W.numels(W.c1_ragged()) + [5, 70001, 3]
_ctr = [0]


def _group(n, dtype, flags=0, opt="adamw"):
    _ctr[0] += 1
    name = f"cmb{os.getpid()}_{_ctr[0]}"
    g = harness.VirtualGroup(NUMEL, n, 0, dtype, 1 << 20, name, 2, cm.CM_SHADOW_HOST, flags, 0, opt=opt)
    g._shm = name
    return g


def _close(g):
    g.sync()
    g.finalize()
    for r in range(g.n):
        cm.unlink_shadow(g._shm, r)


@pytest.mark.parametrize("opt", ["adamw", "sgd"])
@pytest.mark.parametrize("zero1", [False, True])
@pytest.mark.parametrize("dtype", [cm.CM_F32, cm.CM_BF16])
@pytest.mark.parametrize("n", [1, 2, 4])
def test_bucket_steps_bit_exact(n, dtype, zero1, opt):
    g = _group(n, dtype, cm.CM_FLAG_ZERO1 if zero1 else 0, opt)
    plan = O.Plan(NUMEL, 1 << 20, 4 if dtype == cm.CM_F32 else 2, n)
    if opt == "sgd":
        hp_o = dict(lr=W.HP_SGD["lr"], momentum=W.HP_SGD["momentum"], wd=W.HP_SGD["weight_decay"])
    else:
        hp_o = dict(lr=W.HP["lr"], b1=W.HP["beta1"], b2=W.HP["beta2"], eps=W.HP["eps"], wd=W.HP["weight_decay"])
    ref = O.Run(plan, seed=0, dtype=dtype, gscale=W.GRAD_SCALE, hp=hp_o, opt=opt)
    nb = g.n_buckets
    assert nb >= 3
    try:
        for t in range(5):
            g.gen()
            # all-reduce bucket by bucket (in reverse, as backward produces them); each
            # bucket's step right behind it, except every third one left to cm_apply_step
            for b in reversed(range(nb)):
                for r in g.ranks:
                    r.ctx.allreduce_multicast(b, t, g.stream)
                if b % 3 != 1:
                    for r in g.ranks:
                        if opt == "sgd":
                            r.ctx.apply_bucket_sgd(b, t + 1, stream=g.stream, **g.hp)
                        else:
                            r.ctx.apply_bucket(b, t + 1, stream=g.stream, **g.hp)
            g.apply()
            g.shadow()
            g.t += 1
            ref.step()
            g.sync()
            for r in g.ranks:
                if not zero1:
                    np.testing.assert_array_equal(bits(t2np(r.grad)), bits(ref.R), err_msg=f"R t {t}")
                np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p), err_msg=f"p rank {r.rank} t {t}")
                if not zero1:
                    np.testing.assert_array_equal(bits(t2np(r.m)), bits(ref.m), err_msg=f"m t {t}")
                    np.testing.assert_array_equal(bits(t2np(r.v)), bits(ref.v), err_msg=f"v t {t}")
                assert r.ctx.verify_ex(cm.CM_VERIFY_SHADOW | cm.CM_VERIFY_HOST, g.stream) == (cm.CM_OK, -1, None)
            np.testing.assert_array_equal(bits(ring_flat(g, t % 2)), bits(ref.T), err_msg=f"tap t {t}")
            sp, sm, sv = shadow_flat(g, (t + 1) & 1)
            np.testing.assert_array_equal(bits(sp), bits(ref.sp))
            np.testing.assert_array_equal(bits(sm), bits(ref.sm))
    finally:
        _close(g)


def test_bucket_step_errors():
    g = _group(2, cm.CM_F32)
    try:
        c = g.ranks[0].ctx
        g.gen()
        with pytest.raises(cm.CMError) as e:
            c.apply_bucket(0, 1, stream=g.stream)                 # bucket not all-reduced yet
        assert e.value.status == cm.CM_ERR_STATE
        for r in g.ranks:
            r.ctx.allreduce_multicast(0, 0, g.stream)
        c.apply_bucket(0, 1, stream=g.stream)
        with pytest.raises(cm.CMError) as e:
            c.apply_bucket(0, 1, stream=g.stream)                 # twice
        assert e.value.status == cm.CM_ERR_STATE
        for r in g.ranks:
            r.ctx.allreduce_multicast(1, 0, g.stream)
        with pytest.raises(cm.CMError) as e:
            c.apply_bucket(1, 1, lr=2e-3, stream=g.stream)        # other hyper-parameters
        assert e.value.status == cm.CM_ERR_STATE
        with pytest.raises(cm.CMError) as e:
            c.apply_bucket(1, 2, stream=g.stream)                 # wrong step
        assert e.value.status == cm.CM_ERR_STATE
    finally:
        _close(g)


@pytest.mark.parametrize("zero1", [False, True])
def test_restore_after_partial_bucket_steps(zero1):
    """A kill in the middle of backward with per-bucket steps: some buckets of step 4 already
    updated p (and, ZeRO-1, pushed it to every rank) when the trainer dies.  Restore must
    return step 3 and the run continue bit-exact vs the oracle's uninterrupted run."""
    n = 2
    g = _group(n, cm.CM_F32, cm.CM_FLAG_ZERO1 if zero1 else 0)
    plan = O.Plan(NUMEL, 1 << 20, 4, n)
    hp_o = dict(lr=W.HP["lr"], b1=W.HP["beta1"], b2=W.HP["beta2"], eps=W.HP["eps"], wd=W.HP["weight_decay"])
    ref = O.Run(plan, seed=0, gscale=W.GRAD_SCALE, hp=hp_o)
    try:
        for _ in range(3):
            g.step()
            ref.step()
        g.gen()
        for b in reversed(range(g.n_buckets)):
            for r in g.ranks:
                r.ctx.allreduce_multicast(b, 3, g.stream)
        for b in range(g.n_buckets // 2 + 1):
            for r in g.ranks:
                r.ctx.apply_bucket(b, 4, stream=g.stream, **g.hp)
        g.sync()
        assert [r.ctx.restore(g.stream) for r in g.ranks] == [3, 3]
        g.t = 3
        for _ in range(3):
            g.step()
            ref.step()
        g.sync()
        for r in g.ranks:
            np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p))
            if not zero1:
                np.testing.assert_array_equal(bits(t2np(r.m)), bits(ref.m))
                np.testing.assert_array_equal(bits(t2np(r.v)), bits(ref.v))
            assert r.ctx.verify_ex(cm.CM_VERIFY_ALL, g.stream) == (cm.CM_OK, -1, None)
    finally:
        _close(g)
