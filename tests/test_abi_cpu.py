"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/cm.h
declares, plans buckets exactly like the oracle, and fails loudly (no CPU fallback)."""
import re
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2507_13522_b200 import cm
from paper_2507_13522_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "cm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cm_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_six_paper_calls():
    d = _declared()
    for name in ("cm_init", "cm_register_buckets", "cm_allreduce_multicast", "cm_apply_step",
                 "cm_shadow_apply", "cm_restore"):
        assert name in d


def test_library_exports_every_declared_symbol():
    L = cm.lib()
    declared = _declared()
    assert sorted(cm.EXPORTS) == declared
    for name in declared:
        assert hasattr(L, name), name


def test_plan_matches_oracle_random():
    rng = np.random.default_rng(11)
    for _ in range(200):
        nt = int(rng.integers(1, 30))
        numel = [int(x) for x in rng.integers(1, 3000, nt)]
        cap = int(rng.integers(8, 30000))
        dt = int(rng.integers(0, 2))
        n = int(rng.choice([1, 2, 4, 8]))
        tot, nb, offs = cm.plan_buckets(numel, dt, cap, n)
        ref = O.Plan(numel, cap, 4 if dt == 0 else 2, n)
        assert tot == ref.total and nb == ref.n_buckets
        assert offs == list(ref.tensor_off)
        table = cm.plan_bucket_table(numel, dt, cap, n)
        assert [t[0] for t in table] == list(ref.bucket_off)
        assert [t[1] for t in table] == list(ref.bucket_padded)
        assert [t[2] for t in table] == list(ref.bucket_used)


def test_plan_paper_models():
    tot, nb, _ = cm.plan_buckets(W.numels(W.gpt2_small()), cm.CM_F32, W.CAP_BYTES, 8)
    assert (tot, nb) == (124439808, 17)
    tot, nb, _ = cm.plan_buckets(W.numels(W.llama3_8b()), cm.CM_BF16, W.CAP_BYTES, 8)
    assert (tot, nb) == (8030261248, 226)


def test_plan_rejects_bad_tables():
    for numel, dt, cap, n in (([], 0, 100, 1), ([0], 0, 100, 1), ([5], 0, 0, 1), ([5], 7, 100, 1),
                              ([5], 0, 100, 9), ([5], 0, 100, 0)):
        with pytest.raises(cm.CMError) as e:
            cm.plan_buckets(numel, dt, cap, n)
        assert e.value.status in (cm.CM_ERR_CONFIG, cm.CM_ERR_ARG)


def test_init_rejects_bad_config_before_touching_cuda():
    for kw in (dict(world_size=0, rank=0), dict(world_size=9, rank=0), dict(world_size=2, rank=2),
               dict(world_size=2, rank=0, ring_depth=1)):
        args = dict(world_size=2, rank=0, device=0, ring_depth=2)
        args.update(kw)
        with pytest.raises(cm.CMError) as e:
            cm.Context(args["world_size"], args["rank"], 0, args["ring_depth"])
        assert e.value.status == cm.CM_ERR_CONFIG


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(cm.CMError) as e:
        cm.Context(1, 0, 0, 2, shm_name="nofallback")
    assert e.value.status == cm.CM_ERR_CUDA
