"""Edge-case parity of the CUDA path and the non-finite contract.

- Hand-built inputs through the whole path (reduce, tap, AdamW, shadow), bitwise vs the
  oracle: subnormal gradients and subnormal second moments (reading R17: no FTZ/DAZ, the
  IEEE division / square root slow paths), exact +-0 sums (R3: the sum is seeded with g_0),
  the rank-order pin [1, 2^24, -2^24] at n = 3 (R2), large finite values.
- Near-overflow sums (up to 2^127 magnitudes): R bitwise vs the oracle, the overflowing
  element reported as non-finite with its flat index.
- inf / NaN gradients and an AdamW state overflow ("non-finite input ->
  numeric error"; reading R16): CM_ERR_INVARIANT with the flat index (cm_check,
  cm_verify_ex), the shadow does not apply the flagged step (device side: the calls are all
  issued before the flagging kernel runs), cm_restore returns the last finite step, and
  training continues bit-exact vs the oracle's run that never saw the bad values.
"""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2507_13522_b200 import cm, harness
from paper_2507_13522_b200 import workloads as W
from tests.gpu_util import bits, flat_to_local, ring_flat, shadow_flat, t2np

pytestmark = pytest.mark.gpu

HP_O = dict(lr=W.HP["lr"], b1=W.HP["beta1"], b2=W.HP["beta2"], eps=W.HP["eps"], wd=W.HP["weight_decay"])
NUMEL = [70000, 3, 262145, 17, 5000]
CAP = 1 << 20
_ctr = [0]


def _group(n, dtype, D=2, K=1):
    _ctr[0] += 1
    name = f"cme{os.getpid()}_{_ctr[0]}"
    g = harness.VirtualGroup(NUMEL, n, 0, dtype, CAP, name, D, cm.CM_SHADOW_HOST, 0, 0, persist_every=K)
    g._shm = name
    return g


def _close(g):
    g.sync()
    g.finalize()
    for r in range(g.n):
        cm.unlink_shadow(g._shm, r)


def f32b(x):
    return np.float32(x).view(np.uint32)


def bf(x):
    """bf16 bits of an exactly representable value."""
    u = int(np.float32(x).view(np.uint32))
    assert u & 0xFFFF == 0, x
    return np.uint16(u >> 16)


def _set(g, grads):
    for r, a in zip(g.ranks, grads):
        if a.dtype == np.uint16:
            r.grad.view(torch.int16).copy_(torch.from_numpy(a.view(np.int16)))
        else:
            r.grad.copy_(torch.from_numpy(a))
    torch.cuda.synchronize()


def _hold(g, ms=60):
    """Keep the training stream busy while the host enqueues a whole iteration, so that every
    call is issued before the kernel that flags a bad value runs (the report is read by the
    host at each call; this makes the device-side handling -- the shadow skipping the flagged
    step -- what the test exercises)."""
    with torch.cuda.stream(g.stream):
        torch.cuda._sleep(int(ms * 2e6))


def _edge_grads(plan, n, dtype, t, rng):
    """Generated grads for iteration t with edge patterns written over the same used
    elements every iteration (so the moments of those elements stay in the edge regime)."""
    gs = [O.gen_grads(plan, 0, r, t, dtype, W.GRAD_SCALE) for r in range(n)]
    used = np.flatnonzero(plan.used_mask())
    pos = np.random.default_rng(11).choice(used, 64 * 8, replace=False).reshape(8, 64)
    if dtype == O.F32:
        pats = [
            [0.0] * n,                                           # +0 sum
            [-0.0] * n,                                          # -0 + -0 = -0 (seeded with g_0)
            [-0.0] + [0.0] * (n - 1),                            # -0 + +0 = +0
            [2.0 ** -140] + [-(2.0 ** -145)] * (n - 1),          # subnormal operands and sums
            [2.0 ** -149] * n,                                   # smallest subnormal
            [2.0 ** -64] * n,                                    # g*g = 2^-128 (subnormal), v subnormal
            ([1.0, 2.0 ** 24, -(2.0 ** 24)] + [0.0] * 5)[:n],   # rank order: (1 + 2^24) - 2^24 = 0
            [2.0 ** 60, -(2.0 ** 59)] + [2.0 ** 40] * (n - 2),   # large, finite g*g
        ]
        for pat, ps in zip(pats, pos):
            for r in range(n):
                gs[r][ps] = np.float32(pat[r])
    else:
        pats = [
            [0.0] * n, [-0.0] * n, [-0.0] + [0.0] * (n - 1),
            [2.0 ** -133] + [-(2.0 ** -130)] * (n - 1),          # bf16 subnormals
            [2.0 ** -133] * n,
            [2.0 ** -64] * n,
            ([1.0, 2.0 ** 24, -(2.0 ** 24)] + [0.0] * 5)[:n],
            [2.0 ** 60, -(2.0 ** 59)] + [2.0 ** 40] * (n - 2),
        ]
        for pat, ps in zip(pats, pos):
            for r in range(n):
                gs[r][ps] = bf(pat[r])
    return gs


@pytest.mark.parametrize("dtype", [cm.CM_F32, cm.CM_BF16])
@pytest.mark.parametrize("n", [2, 3])
def test_edge_values_full_path_bit_exact(n, dtype):
    plan = O.Plan(NUMEL, CAP, 4 if dtype == cm.CM_F32 else 2, n)
    ref = O.Run(plan, seed=0, dtype=dtype, gscale=W.GRAD_SCALE, hp=HP_O)
    g = _group(n, dtype)
    rng = np.random.default_rng(7)
    try:
        for t in range(6):
            grads = _edge_grads(plan, n, dtype, t, rng)
            _set(g, grads)
            g.step(gen=False)
            ref.step(grads=grads)
            g.sync()
            for r in g.ranks:
                np.testing.assert_array_equal(bits(t2np(r.grad)), bits(ref.R), err_msg=f"R t {t}")
                for nm, a, b in (("p", r.p, ref.p), ("m", r.m, ref.m), ("v", r.v, ref.v)):
                    np.testing.assert_array_equal(bits(t2np(a)), bits(b), err_msg=f"{nm} rank {r.rank} t {t}")
            np.testing.assert_array_equal(bits(ring_flat(g, t % 2)), bits(ref.T), err_msg=f"tap t {t}")
            sp, sm, sv = shadow_flat(g, (t + 1) & 1)
            for nm, a, b in (("sp", sp, ref.sp), ("sm", sm, ref.sm), ("sv", sv, ref.sv)):
                np.testing.assert_array_equal(bits(a), bits(b), err_msg=f"shadow {nm} t {t}")
            for r in g.ranks:
                assert r.ctx.verify_ex(cm.CM_VERIFY_ALL, g.stream) == (cm.CM_OK, -1, None)
                assert r.ctx.info().nonfinite_step == -1
        # the patterns really reached the interesting regimes
        v = ref.v[ref.v != 0]
        assert np.any(np.abs(v) < np.finfo(np.float32).tiny), "no subnormal second moment"
        assert np.any(ref.R.view(np.uint32 if dtype == cm.CM_F32 else np.uint16) ==
                      (0x80000000 if dtype == cm.CM_F32 else 0x8000)), "no -0 sum"
    finally:
        _close(g)


@pytest.mark.parametrize("dtype", [cm.CM_F32, cm.CM_BF16])
def test_near_overflow_reduce_bit_exact_and_flagged(dtype):
    n = 2
    plan = O.Plan(NUMEL, CAP, 4 if dtype == cm.CM_F32 else 2, n)
    g = _group(n, dtype)
    try:
        gs = [O.gen_grads(plan, 0, r, 0, dtype, W.GRAD_SCALE) for r in range(n)]
        used = np.flatnonzero(plan.used_mask())
        rng = np.random.default_rng(3)
        ps = rng.choice(used, 40, replace=False)
        big = [(1.5 * 2.0 ** 127, -(2.0 ** 127)), (2.0 ** 127, -(2.0 ** 126)), (-(2.0 ** 127), -(2.0 ** 126)),
               (1.5 * 2.0 ** 126, 1.5 * 2.0 ** 126)]
        for k, i in enumerate(ps[:-1]):
            a, b = big[k % len(big)]
            for r, x in enumerate((a, b)):
                gs[r][i] = np.float32(x) if dtype == cm.CM_F32 else bf(x)
        over = int(ps[-1])                       # 2^127 + 2^127 overflows to +inf
        for r in range(n):
            gs[r][over] = np.float32(2.0 ** 127) if dtype == cm.CM_F32 else bf(2.0 ** 127)
        _set(g, gs)
        _hold(g)
        g.allreduce(t=0)
        g.sync()
        R = O.reduce_f32(gs) if dtype == cm.CM_F32 else O.reduce_bf16(gs)
        assert np.isinf(R.view(np.float32)[over]) if dtype == cm.CM_F32 else (R[over] == 0x7F80)
        for r in g.ranks:
            np.testing.assert_array_equal(bits(t2np(r.grad)), bits(R))
        owner, _ = flat_to_local(g.ranks, [over])
        info = g.ranks[int(owner[0])].ctx.info()
        assert (info.nonfinite_step, info.nonfinite_index) == (1, over)
        assert g.ranks[int(owner[0])].ctx.check() == (cm.CM_ERR_INVARIANT, 1, over)
    finally:
        _close(g)


@pytest.mark.parametrize("dtype", [cm.CM_F32, cm.CM_BF16])
@pytest.mark.parametrize("kind", ["nan", "inf", "adam_overflow"])
def test_nonfinite_is_refused_and_restore_recovers(kind, dtype):
    n, D, K = 2, 4, 2
    plan = O.Plan(NUMEL, CAP, 4 if dtype == cm.CM_F32 else 2, n)
    ref = O.Run(plan, seed=0, dtype=dtype, gscale=W.GRAD_SCALE, hp=HP_O)
    g = _group(n, dtype, D=D, K=K)
    try:
        for _ in range(3):
            g.step()
            ref.step()
        g.sync()
        # one bad value in rank 1's gradients, at an element of rank 0's shard
        owner, _ = flat_to_local(g.ranks, np.flatnonzero(plan.used_mask()))
        i = int(np.flatnonzero(plan.used_mask())[np.flatnonzero(owner == 0)[1234]])
        g.gen()
        g.sync()
        bad = {"nan": float("nan"), "inf": float("inf"), "adam_overflow": 2.0 ** 80}[kind]
        if dtype == cm.CM_F32:
            g.ranks[1].grad[i] = bad
        else:
            bits16 = {"nan": 0x7FC0, "inf": 0x7F80, "adam_overflow": int(bf(2.0 ** 80))}[kind]
            g.ranks[1].grad.view(torch.int16)[i] = int(np.uint16(bits16).view(np.int16))
        torch.cuda.synchronize()
        _hold(g)
        g.allreduce()
        g.apply()
        g.shadow()
        g.t += 1
        g.sync()
        for r in g.ranks:
            st, mis, what = r.ctx.verify_ex(cm.CM_VERIFY_ALL, g.stream)
            assert (st, mis, what) == (cm.CM_ERR_INVARIANT, i, "nonfinite"), (r.rank, st, mis, what)
            info = r.ctx.info()
            assert (info.nonfinite_step, info.nonfinite_index) == (4, i)
            assert info.shadow_step in (3, 4)
        assert g.ranks[0].ctx.info().shadow_step == 3      # the owner's shadow never applied step 4
        assert g.ranks[0].ctx.check() == (cm.CM_ERR_INVARIANT, 4, i)
        steps = [r.ctx.restore(g.stream) for r in g.ranks]
        assert steps == [3, 3]
        for r in g.ranks:
            assert r.ctx.info().nonfinite_step == -1
            assert r.ctx.check() == (cm.CM_OK, -1, -1)
        g.t = 3
        for _ in range(3):
            g.step()
            ref.step()
        g.sync()
        for r in g.ranks:
            for nm, a, b in (("p", r.p, ref.p), ("m", r.m, ref.m), ("v", r.v, ref.v)):
                np.testing.assert_array_equal(bits(t2np(a)), bits(b), err_msg=f"{nm} rank {r.rank}")
            assert r.ctx.verify_ex(cm.CM_VERIFY_ALL, g.stream) == (cm.CM_OK, -1, None)
    finally:
        _close(g)
