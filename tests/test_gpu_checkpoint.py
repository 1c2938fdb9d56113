"""The checkpoint bytes that carry the paper's claim, checked where they land.

PAPER.md:605 (sec 6.5): the shadow's replica must be identical to the training replica;
PAPER.md:601: the recovery methodology -- halt and restore during every second iteration,
compare with an uninterrupted run.  SPEC.md:433-435, 588-596, 634-635.

- cm_verify_ex can fail: one flipped bit in the training p/m/v, in a host snapshot half or in
  a tapped ring slot is found, with its flat index (negative tests of the comparator).
- GPT-2 small at full size in bench.py's configuration (host shadow, K=8 snapshots, ring
  depth D=16, staged tap, coalesced copy-engine/SM drains): every iteration the host log
  alone (snapshot + ring roll-forward) reproduces the training state bitwise, the ring slot
  equals the reduced gradients, and sampled ring / snapshot elements (plus every bucket edge)
  equal the oracle; then a hard kill, attach, restore, and 100 more iterations vs the oracle.
- Halt-and-restore every second iteration for 100 iterations (three kill points), every
  completed iteration compared element by element with the oracle's uninterrupted run.
"""
import ctypes as C
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2507_13522_b200 import cm, harness
from paper_2507_13522_b200 import workloads as W
from tests.gpu_util import bits, flat_to_local, flip_host_bit, host_view, local_to_flat, ring_flat, t2np

pytestmark = pytest.mark.gpu

HP_O = dict(lr=W.HP["lr"], b1=W.HP["beta1"], b2=W.HP["beta2"], eps=W.HP["eps"], wd=W.HP["weight_decay"])
_ctr = [0]


def _name():
    _ctr[0] += 1
    return f"cmk{os.getpid()}_{_ctr[0]}"


def group(numel, n, cap=1 << 20, D=4, K=4, flags=0, name=None, dtype=cm.CM_F32):
    name = name or _name()
    g = harness.VirtualGroup(numel, n, 0, dtype, cap, name, D, cm.CM_SHADOW_HOST, flags, 0, persist_every=K)
    g._shm = name
    return g


def close(g, unlink=True):
    g.sync()
    g.finalize()
    if unlink:
        for r in range(g.n):
            cm.unlink_shadow(g._shm, r)


def all_ok(g):
    for r in g.ranks:
        st, mis, what = r.ctx.verify_ex(cm.CM_VERIFY_ALL, g.stream)
        assert (st, mis, what) == (cm.CM_OK, -1, None), (r.rank, st, mis, what)


@pytest.mark.parametrize("n", [1, 2])
def test_verify_finds_every_single_bit_flip(n):
    """Negative tests: the comparator reports the exact flat index of one flipped bit in the
    training state, in the host snapshot the restore would start from, and in a ring slot."""
    numel = W.numels(W.c1_ragged())
    g = group(numel, n, D=4, K=4)
    try:
        for _ in range(6):                        # snapshots at 0 and 4; ring holds steps 5, 6
            g.step()
        g.sync()
        all_ok(g)
        rng = np.random.default_rng(1)
        for r in g.ranks:
            info = r.ctx.info()
            assert info.host_half_step[0] in (0, 4) and info.host_half_step[1] in (0, 4)
            L = info.shard_numel
            # (1) training p, m, v on the device: SHADOW scope (and HOST) finds it
            for arr, name in ((r.p, "p"), (r.m, "m"), (r.v, "v")):
                j = int(rng.integers(0, L))
                i = local_to_flat(r, j)
                w = arr.view(torch.int32)
                w[i] ^= 1 << 3
                torch.cuda.synchronize()
                st, mis, what = r.ctx.verify_ex(cm.CM_VERIFY_SHADOW, g.stream)
                assert (st, mis, what) == (cm.CM_ERR_INVARIANT, i, name)
                st, mis, what = r.ctx.verify_ex(cm.CM_VERIFY_HOST, g.stream)
                assert (st, mis, what) == (cm.CM_ERR_INVARIANT, i, name)
                w[i] ^= 1 << 3
                torch.cuda.synchronize()
            # (2) the host snapshot half at step 4 (the restore source; rolled forward to 6)
            half = 0 if info.host_half_step[0] == 4 else 1
            ptrs = r.ctx.shadow_view(half)
            for a, name in enumerate(("p", "m", "v")):
                j = int(rng.integers(0, L))
                i = local_to_flat(r, j)
                flip_host_bit(ptrs[a], j, bit=5)
                st, mis, what = r.ctx.verify_ex(cm.CM_VERIFY_HOST, g.stream)
                # a wrong m (or v) also changes the rolled-forward p of that element, which
                # sorts first (p < m < v at one index)
                assert st == cm.CM_ERR_INVARIANT and mis == i and what in ("p", name), (name, mis, what)
                assert r.ctx.verify_ex(cm.CM_VERIFY_SHADOW, g.stream)[0] == cm.CM_OK   # HBM shadow untouched
                flip_host_bit(ptrs[a], j, bit=5)
            # (3) a ring slot: iteration 5's gradients (step 6) -- RING and HOST scopes
            j = int(rng.integers(0, L))
            i = local_to_flat(r, j)
            slot = (6 - 1) % 4
            flip_host_bit(r.ctx.ring_view(slot), j, bit=20)
            assert r.ctx.verify_ex(cm.CM_VERIFY_RING, g.stream) == (cm.CM_ERR_INVARIANT, i, "ring")
            st, mis, what = r.ctx.verify_ex(cm.CM_VERIFY_HOST, g.stream)
            assert st == cm.CM_ERR_INVARIANT and mis == i
            flip_host_bit(r.ctx.ring_view(slot), j, bit=20)
            # (4) an older ring slot inside the roll-forward window (step 5)
            flip_host_bit(r.ctx.ring_view((5 - 1) % 4), j, bit=20)
            assert r.ctx.verify_ex(cm.CM_VERIFY_RING, g.stream)[0] == cm.CM_OK
            st, mis, what = r.ctx.verify_ex(cm.CM_VERIFY_HOST, g.stream)
            assert st == cm.CM_ERR_INVARIANT and mis == i
            flip_host_bit(r.ctx.ring_view((5 - 1) % 4), j, bit=20)
        all_ok(g)
    finally:
        close(g)


def _sample(plan, seed=0, k=1 << 14):
    rng = np.random.default_rng(seed)
    idx = rng.choice(plan.total, k, replace=False)
    edges = np.concatenate([plan.bucket_off, plan.bucket_off + plan.bucket_padded - 1])
    return np.unique(np.concatenate([idx, edges])).astype(np.int64)


@pytest.mark.parametrize("n", [1, 2])
def test_gpt2_bench_config_host_log_and_hard_restore(n):
    """GPT-2 small, full size, bench.py's shadow configuration (HOST, K=8, D=16, staged tap,
    automatic drain policy with coalesced drains).  Every iteration: CM_VERIFY_ALL (the host
    log alone rebuilds the training state; the ring slot equals the reduced gradients) and
    sampled + bucket-edge ring elements vs the oracle's R; every persisted snapshot sampled vs
    the oracle.  Then a hard kill with the shadow one step behind, attach, restore (rolls
    forward to the last tapped step), 100 more iterations, sampled vs the oracle."""
    numel = W.numels(W.gpt2_small())
    plan = O.Plan(numel, W.CAP_BYTES, 4, n)
    idx = _sample(plan)
    used = plan.used_mask()[idx]
    name = _name()
    D, K, T0 = 16, 8, 24
    g = group(numel, n, cap=W.CAP_BYTES, D=D, K=K, name=name)
    owner, local = flat_to_local(g.ranks, idx)
    try:
        L = g.ranks[0].ctx.info().shard_numel
        for t in range(T0):
            g.step()
            g.sync()
            all_ok(g)
            p, m, v, R = O.run_sample(0, n, O.F32, W.GRAD_SCALE, t + 1, idx, used, **HP_O)
            ring = np.empty(len(idx), np.float32)
            for r in g.ranks:
                sel = owner == r.rank
                ring[sel] = host_view(r.ctx.ring_view(t % D), L, np.float32)[local[sel]]
            np.testing.assert_array_equal(bits(ring), bits(R), err_msg=f"ring t {t}")
            if (t + 1) % K == 0:                 # a snapshot was persisted at step t+1
                for r in g.ranks:
                    info = r.ctx.info()
                    half = [h for h in (0, 1) if info.host_half_step[h] == t + 1]
                    assert half, (t, list(info.host_half_step))
                    ptrs = r.ctx.shadow_view(half[0])
                    sel = owner == r.rank
                    for a, ref in zip(ptrs, (p, m, v)):
                        np.testing.assert_array_equal(bits(host_view(a, L, np.float32)[local[sel]]),
                                                      bits(ref[sel]), err_msg=f"snapshot t {t}")
        g.step(shadow=False)                     # iteration T0: tapped, not applied by the shadow
        g.sync()
        for r in g.ranks:
            assert r.ctx.info().shadow_step == T0
        close(g, unlink=False)                   # the process "dies": only /dev/shm survives
        del g
        torch.cuda.empty_cache()
        g2 = group(numel, n, cap=W.CAP_BYTES, D=D, K=K, name=name, flags=cm.CM_FLAG_ATTACH)
        try:
            for r in g2.ranks:
                r.p.fill_(float("nan"))
                r.m.fill_(float("nan"))
            torch.cuda.synchronize()
            steps = [r.ctx.restore(g2.stream) for r in g2.ranks]
            assert steps == [T0 + 1] * n
            for r in g2.ranks:                   # (the grad buffer holds nothing yet: no RING scope)
                st = r.ctx.verify_ex(cm.CM_VERIFY_SHADOW | cm.CM_VERIFY_HOST, g2.stream)
                assert st == (cm.CM_OK, -1, None), st
            g2.t = T0 + 1
            for _ in range(100):
                g2.step()
            g2.sync()
            all_ok(g2)
            p, m, v, R = O.run_sample(0, n, O.F32, W.GRAD_SCALE, T0 + 101, idx, used, **HP_O)
            for r in g2.ranks:
                ti = torch.from_numpy(idx).to(r.p.device)
                np.testing.assert_array_equal(bits(r.p[ti].cpu().numpy()), bits(p))
                np.testing.assert_array_equal(bits(r.m[ti].cpu().numpy()), bits(m))
                np.testing.assert_array_equal(bits(r.v[ti].cpu().numpy()), bits(v))
                np.testing.assert_array_equal(bits(r.grad[ti].cpu().numpy()), bits(R))
        finally:
            close(g2)
    finally:
        for r in range(n):
            cm.unlink_shadow(name, r)


@pytest.mark.parametrize("K,D", [(1, 2), (2, 4), (4, 6)])
def test_halt_and_restore_every_second_iteration_for_100(K, D):
    """PAPER.md:601 (sec 6.5): "we halt and restore model training during every second
    iteration for 100 iterations".  Kill points rotate: mid all-reduce (restore
    to t), after the training step but before the shadow step (roll forward to t+1), after
    the shadow step (t+1).  The killed replica's state is poisoned with NaN.  Every completed
    iteration: R, train p/m/v of every rank and the tap ring equal the oracle's
    uninterrupted run element by element."""
    numel = W.numels(W.c1())
    n = 2
    g = group(numel, n, D=D, K=K)
    plan = O.Plan(numel, 1 << 20, 4, n)
    ref = O.Run(plan, seed=0, gscale=W.GRAD_SCALE, hp=HP_O)
    kills = 0
    try:
        t = 0
        while t < 100:
            if t % 2 == 1:
                point = kills % 3
                kills += 1
                if point == 0:                      # mid all-reduce
                    g.gen()
                    for b in range(g.n_buckets // 2 + 1):
                        for r in g.ranks:
                            r.ctx.allreduce_multicast(b, t, g.stream)
                    expect = t
                else:
                    g.gen()
                    g.allreduce()
                    g.apply()
                    if point == 2:
                        g.shadow()
                    expect = t + 1
                g.sync()
                for r in g.ranks:
                    r.p.fill_(float("nan")); r.m.fill_(float("nan")); r.v.fill_(float("nan"))
                torch.cuda.synchronize()
                steps = [r.ctx.restore(g.stream) for r in g.ranks]
                assert steps == [expect] * n, (t, point, steps)
                if expect == t + 1:                 # iteration t survived the kill
                    ref.step()
                    t += 1
                g.t = t
                for r in g.ranks:
                    np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p), err_msg=f"restored p t {t}")
                    np.testing.assert_array_equal(bits(t2np(r.m)), bits(ref.m), err_msg=f"restored m t {t}")
                    np.testing.assert_array_equal(bits(t2np(r.v)), bits(ref.v), err_msg=f"restored v t {t}")
                if t >= 100:
                    break
            g.step()
            ref.step()
            g.sync()
            for r in g.ranks:
                np.testing.assert_array_equal(bits(t2np(r.grad)), bits(ref.R), err_msg=f"R t {t}")
                for nm, a, b in (("p", r.p, ref.p), ("m", r.m, ref.m), ("v", r.v, ref.v)):
                    np.testing.assert_array_equal(bits(t2np(a)), bits(b), err_msg=f"{nm} rank {r.rank} t {t}")
            np.testing.assert_array_equal(bits(ring_flat(g, t % D)), bits(ref.T), err_msg=f"tap t {t}")
            t += 1
        assert kills >= 45
        for r in g.ranks:          # (the run may end right after a restore: no RING scope then)
            assert r.ctx.verify_ex(cm.CM_VERIFY_SHADOW | cm.CM_VERIFY_HOST, g.stream) == (cm.CM_OK, -1, None)
    finally:
        close(g)


def test_c1_100_iterations_full_compare():
    """100 iterations of C1 (n=2, 2^20 fp32, 4 buckets), every element of R, the
    tap ring, train p/m/v and the host shadow halves vs the oracle every iteration."""
    numel = W.numels(W.c1())
    n = 2
    g = group(numel, n, D=2, K=1)
    plan = O.Plan(numel, 1 << 20, 4, n)
    ref = O.Run(plan, seed=0, gscale=W.GRAD_SCALE, hp=HP_O)
    from tests.gpu_util import shadow_flat
    try:
        for t in range(100):
            g.step()
            ref.step()
            g.sync()
            np.testing.assert_array_equal(bits(ring_flat(g, t % 2)), bits(ref.T), err_msg=f"tap t {t}")
            for r in g.ranks:
                np.testing.assert_array_equal(bits(t2np(r.grad)), bits(ref.R), err_msg=f"R t {t}")
                for nm, a, b in (("p", r.p, ref.p), ("m", r.m, ref.m), ("v", r.v, ref.v)):
                    np.testing.assert_array_equal(bits(t2np(a)), bits(b), err_msg=f"{nm} t {t}")
            sp, sm, sv = shadow_flat(g, (t + 1) & 1)
            for nm, a, b in (("sp", sp, ref.sp), ("sm", sm, ref.sm), ("sv", sv, ref.sv)):
                np.testing.assert_array_equal(bits(a), bits(b), err_msg=f"shadow {nm} t {t}")
            if t % 10 == 9:
                all_ok(g)
    finally:
        close(g)


def test_surviving_segment_is_never_replaced_implicitly():
    """a fresh context must not delete a surviving shadow segment (the restore
    source after a hard kill).  Without CM_FLAG_OVERWRITE cm_connect refuses (CM_ERR_STATE);
    CM_FLAG_ATTACH attaches; CM_FLAG_OVERWRITE starts fresh on purpose."""
    numel = W.numels(W.c1())
    g = group(numel, 1, D=2, K=1)
    name = g._shm
    try:
        g.step()
        close(g, unlink=False)
        r = harness.Rank(numel, 1, 0, 0, cm.CM_F32, 1 << 20, name, 2, cm.CM_SHADOW_HOST, 0, overwrite=False)
        with pytest.raises(cm.CMError) as e:
            r.ctx.connect([r.blob])
        assert e.value.status == cm.CM_ERR_STATE
        r.ctx.finalize()
        assert os.path.exists(f"/dev/shm/{name}.r0")
        r2 = harness.Rank(numel, 1, 0, 0, cm.CM_F32, 1 << 20, name, 2, cm.CM_SHADOW_HOST, cm.CM_FLAG_ATTACH)
        r2.ctx.connect([r2.blob])
        assert r2.ctx.restore(None) == 1
        r2.ctx.finalize()
    finally:
        cm.unlink_shadow(name, 0)


def test_n1_copy_engine_staging_bit_exact():
    """n == 1 ablation "n1_copy_engine": the bucket's copy into the staging half by a copy
    engine instead of a kernel; R, ring, p/m/v and shadow stay bitwise equal to the oracle."""
    numel = W.numels(W.c1_ragged())
    g = group(numel, 1, D=4, K=2)
    for r in g.ranks:
        r.ctx.set_param("n1_copy_engine", 1)
    plan = O.Plan(numel, 1 << 20, 4, 1)
    ref = O.Run(plan, seed=0, gscale=W.GRAD_SCALE, hp=HP_O)
    try:
        for t in range(5):
            g.step()
            ref.step()
            g.sync()
            r = g.ranks[0]
            np.testing.assert_array_equal(bits(t2np(r.p)), bits(ref.p), err_msg=f"p t {t}")
            np.testing.assert_array_equal(bits(t2np(r.v)), bits(ref.v), err_msg=f"v t {t}")
            np.testing.assert_array_equal(bits(ring_flat(g, t % 4)), bits(ref.T), err_msg=f"tap t {t}")
            all_ok(g)
    finally:
        close(g)
