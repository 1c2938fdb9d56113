"""Shadow serving against the oracle (SPEC.md:422-430 serve_checkpoint,
SPEC.md:411-421 consolidate; sec 4.2.4): after a run with host snapshots
every K steps, the consolidated checkpoint fetched from the n shards' host segments --
every shard in parallel, CRC-32 checked -- equals the oracle's p, m, v at that step,
bitwise, and so does the retained previous snapshot, every single tensor, and the
per-tensor model file cm_shadow_export writes.  While
training keeps running (the shadow rewriting halves under the reader), every fetch that
succeeds equals the oracle at the step it names."""
import os
import threading

import numpy as np
import pytest

from oracle import oracle as O
from paper_2507_13522_b200 import cm, harness, serving
from paper_2507_13522_b200 import workloads as W
from tests.gpu_util import bits

pytestmark = pytest.mark.gpu

NUMEL = W.numels(W.c1_ragged()) + [5, 70001, 3]
_ctr = [0]


def _hp_o(opt):
    if opt == "sgd":
        return dict(lr=W.HP_SGD["lr"], momentum=W.HP_SGD["momentum"], wd=W.HP_SGD["weight_decay"])
    return dict(lr=W.HP["lr"], b1=W.HP["beta1"], b2=W.HP["beta2"], eps=W.HP["eps"], wd=W.HP["weight_decay"])


def _group(numel, n, K, D, opt="adamw", dtype=cm.CM_F32, cap=1 << 20, flags=0):
    _ctr[0] += 1
    name = f"cmsv{os.getpid()}_{_ctr[0]}"
    g = harness.VirtualGroup(numel, n, 0, dtype, cap, name, D, cm.CM_SHADOW_HOST, flags, persist_every=K, opt=opt)
    g._shm = name
    return g


def _close(g):
    g.sync()
    g.finalize()
    for r in range(g.n):
        cm.unlink_shadow(g._shm, r)


@pytest.mark.parametrize("n,dtype,opt,flags", [(1, cm.CM_F32, "adamw", 0), (2, cm.CM_F32, "adamw", 0),
                                               (4, cm.CM_BF16, "adamw", 0), (3, cm.CM_F32, "sgd", 0),
                                               (2, cm.CM_BF16, "adamw", cm.CM_FLAG_ZERO1)])
def test_fetch_equals_oracle(n, dtype, opt, flags, tmp_path):
    """flags = CM_FLAG_ZERO1: the trainers hold only their m/v shard, the shadow the same
    shard-local layout; the served model is the same."""
    K, D, T = 2, 3, 5
    g = _group(NUMEL, n, K, D, opt, dtype, flags=flags)
    es = 4 if dtype == cm.CM_F32 else 2
    ref = O.Run(O.Plan(NUMEL, 1 << 20, es, n), seed=0, dtype=dtype, gscale=W.GRAD_SCALE, hp=_hp_o(opt), opt=opt)
    smap = serving.ShardMap(NUMEL, dtype, 1 << 20, n)
    saved = {0: (ref.p.copy(), ref.m.copy(), ref.v.copy())}
    try:
        for t in range(T):
            g.step()
            ref.step()
            saved[t + 1] = (ref.p.copy(), ref.m.copy(), ref.v.copy())
        g.sync()
        assert smap.padded == len(ref.p)
        assert serving.consolidate(g._shm, n) == 4              # snapshots at steps 2 and 4
        for step in (4, 2):                                     # newest, and the retained half
            got_step, got = serving.fetch(g._shm, smap, step=None if step == 4 else step, threads=4,
                                          chunk_elems=100000)
            assert got_step == step
            for k, w in enumerate("pmv"):
                np.testing.assert_array_equal(bits(got[w]), bits(saved[step][k]), err_msg=f"{w} step {step}")
        for i in range(len(NUMEL)):
            _, t_p = serving.fetch_tensor(g._shm, smap, i, what="p")
            lo = smap.tensor_off[i]
            np.testing.assert_array_equal(bits(t_p), bits(saved[4][0][lo:lo + NUMEL[i]]))
        with pytest.raises(cm.CMError) as e:                    # step 3 was never persisted
            serving.fetch(g._shm, smap, step=3)
        assert e.value.status == cm.CM_ERR_STATE
        # the per-tensor model file of the consolidated step (cm_shadow_export)
        path = tmp_path / "model.ckpt"
        assert serving.export(g._shm, NUMEL, dtype, 1 << 20, n, path) == 4
        hdr, recs = serving.read_model_file(path)
        assert hdr["step"] == 4 and len(recs) == len(NUMEL)
        for i, rec in enumerate(recs):
            lo = smap.tensor_off[i]
            for k, w in enumerate("pmv"):
                np.testing.assert_array_equal(bits(rec[w]), bits(saved[4][k][lo:lo + NUMEL[i]]), err_msg=f"{w} {i}")
    finally:
        _close(g)


def test_fetch_while_training_runs():
    """A reader thread fetches the consolidated checkpoint over and over while the group
    trains; the shadow rewrites the older half every K steps under it."""
    n, K, D, T = 2, 2, 3, 24
    numel = [3 << 20, 1 << 20, 12345]
    g = _group(numel, n, K, D, cap=4 << 20)
    ref = O.Run(O.Plan(numel, 4 << 20, 4, n), seed=0, gscale=W.GRAD_SCALE, hp=_hp_o("adamw"))
    smap = serving.ShardMap(numel, cm.CM_F32, 4 << 20, n)
    saved = {0: ref.p.copy()}
    for t in range(T):
        ref.step()
        if (t + 1) % K == 0:
            saved[t + 1] = ref.p.copy()
    got_steps, refused, errors = [], [0], []
    stop = threading.Event()

    def reader():
        while not stop.is_set():
            try:
                step, got = serving.fetch(g._shm, smap, what=("p",), threads=2)
            except cm.CMError as e:
                if e.status != cm.CM_ERR_STATE:
                    errors.append(repr(e))
                    return
                refused[0] += 1
                continue
            if not np.array_equal(bits(got["p"]), bits(saved[step])):
                errors.append(f"step {step}: served bytes differ from the oracle")
                return
            got_steps.append(step)

    th = threading.Thread(target=reader)
    th.start()
    try:
        for t in range(T):
            g.step()
            if t % 4 == 3:
                g.sync()                                   # let the reader see progress
    finally:
        g.sync()
        stop.set()
        th.join()
        _close(g)
    assert not errors, errors
    assert len(got_steps) > 0 and got_steps == sorted(got_steps), got_steps
