"""Model mode: a real model's backward drives the per-bucket all-reduce + tap
through hooks (CheckmateDDP).  Checked against the oracle: after every iteration the
training state equals the oracle's AdamW applied to the gradients the backward produced
(n=1: the all-reduce is the identity), bitwise, and the shadow equals the training state."""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2507_13522_b200 import cm
from paper_2507_13522_b200 import workloads as W

pytestmark = pytest.mark.gpu


def tiny_gpt2():
    from transformers import GPT2Config, GPT2LMHeadModel
    torch.manual_seed(0)
    cfg = GPT2Config(n_layer=2, n_embd=128, n_head=4, n_positions=128, vocab_size=1000)
    cfg._attn_implementation = "sdpa"
    return GPT2LMHeadModel(cfg)


@pytest.mark.parametrize("bucket_step", [False, True])
def test_checkmate_ddp_matches_oracle_adamw_on_model_gradients(bucket_step):
    """bucket_step=True: each bucket's AdamW runs on the comm stream right behind its
    all-reduce, during backward (cm_apply_bucket); same bits."""
    from paper_2507_13522_b200.ddp import CheckmateDDP
    dev = torch.device("cuda", 0)
    model = tiny_gpt2().to(dev)
    name = f"cmddpt{os.getpid()}_{int(bucket_step)}"
    cd = CheckmateDDP(model, 0, 1, 0, cap_bytes=64 << 10, shm_name=name, ring_depth=4, persist_every=2,
                      bucket_step=bucket_step)
    r = cd.r
    numel = [p.numel() for p in cd.params]
    assert len(cd.size) > 3                                # several buckets
    p = r.p.cpu().numpy().copy()
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    gen = torch.Generator(device=dev)
    gen.manual_seed(5)
    try:
        for t in range(4):
            tok = torch.randint(0, 1000, (4, 128), device=dev, generator=gen)
            cd.zero_grad()
            with torch.autocast("cuda", dtype=torch.bfloat16):
                loss = model(tok, labels=tok).loss
            loss.backward()
            torch.cuda.synchronize()
            g = r.grad.cpu().numpy().copy()                # the backward's gradients (n=1: R = g)
            cd.step()
            torch.cuda.synchronize()
            O.adamw(g, O.scalars(t + 1, lr=W.HP["lr"], b1=W.HP["beta1"], b2=W.HP["beta2"], eps=W.HP["eps"],
                                 wd=W.HP["weight_decay"], n=1), p, m, v)
            np.testing.assert_array_equal(r.p.cpu().numpy().view(np.uint32), p.view(np.uint32))
            np.testing.assert_array_equal(r.v.cpu().numpy().view(np.uint32), v.view(np.uint32))
            cd.side.synchronize()
            assert r.ctx.verify_ex(cm.CM_VERIFY_ALL, torch.cuda.current_stream()) == (cm.CM_OK, -1, None)
        # the module's parameters are the flat buffer: a forward after the step sees p
        w = model.transformer.wte.weight
        off = r.tensor_off[0]
        assert w.data_ptr() == r.p[off:].data_ptr()
    finally:
        cd.finalize()
        cm.unlink_shadow(name, 0)


def test_grad_probe_model_parity_n1():
    """The probe-based check used for n > 1 (tests/model_parity.py), here at n=1."""
    from paper_2507_13522_b200.ddp import CheckmateDDP, GradProbe
    from tests.model_parity import check_records, probe_indices
    dev = torch.device("cuda", 0)
    model = tiny_gpt2().to(dev)
    name = f"cmddpp{os.getpid()}"
    cd = CheckmateDDP(model, 0, 1, 0, cap_bytes=64 << 10, shm_name=name, ring_depth=4, persist_every=2)
    cd.probe = GradProbe(cd, probe_indices(cd, 2048))
    gen = torch.Generator(device=dev)
    gen.manual_seed(6)
    try:
        for t in range(3):
            tok = torch.randint(0, 1000, (4, 128), device=dev, generator=gen)
            cd.zero_grad()
            with torch.autocast("cuda", dtype=torch.bfloat16):
                loss = model(tok, labels=tok).loss
            loss.backward()
            cd.step()
        out = check_records([cd.probe.records], 1, W.HP)
        assert out["iterations"] == 3 and out["elements"] >= 2048
    finally:
        cd.finalize()
        cm.unlink_shadow(name, 0)


def test_checkmate_ddp_checkpoint_served():
    """Model mode end to end: after training steps with a snapshot every 2 steps, the
    checkpoint fetched from the host segment (serving.fetch, another code path than the
    trainer's buffers) equals the training state bitwise, and the exported per-tensor model
    file holds every parameter tensor of the module."""
    from paper_2507_13522_b200 import serving
    from paper_2507_13522_b200.ddp import CheckmateDDP
    dev = torch.device("cuda", 0)
    model = tiny_gpt2().to(dev)
    name = f"cmddps{os.getpid()}"
    cd = CheckmateDDP(model, 0, 1, 0, cap_bytes=64 << 10, shm_name=name, ring_depth=4, persist_every=2)
    r = cd.r
    numel = [p.numel() for p in cd.params]
    gen = torch.Generator(device=dev)
    gen.manual_seed(7)
    try:
        for _ in range(4):
            tok = torch.randint(0, 1000, (4, 128), device=dev, generator=gen)
            cd.zero_grad()
            with torch.autocast("cuda", dtype=torch.bfloat16):
                loss = model(tok, labels=tok).loss
            loss.backward()
            cd.step()
        torch.cuda.synchronize()
        cd.side.synchronize()
        smap = serving.ShardMap(numel, cm.CM_F32, 64 << 10, 1)
        step, got = serving.fetch(name, smap)
        assert step == 4
        for w, t in (("p", r.p), ("m", r.m), ("v", r.v)):
            np.testing.assert_array_equal(got[w].view(np.uint32), t.cpu().numpy().view(np.uint32), err_msg=w)
        import tempfile
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "model.ckpt")
            assert serving.export(name, numel, cm.CM_F32, 64 << 10, 1, path) == 4
            hdr, recs = serving.read_model_file(path)
        for prm, rec in zip(cd.params, recs):
            np.testing.assert_array_equal(rec["p"].view(np.uint32),
                                          prm.detach().float().cpu().numpy().ravel().view(np.uint32))
    finally:
        cd.finalize()
        cm.unlink_shadow(name, 0)
