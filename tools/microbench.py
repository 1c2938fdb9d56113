"""Per-kernel microbenchmarks on one GPU (virtual ranks): each kernel timed in isolation
with the library's event timing (cm_timing), reported against its roofline.

  python tools/microbench.py [adamw|tap|tap_ce|ar_virtual|gen|shadow_host|shadow_dev|all]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2507_13522_b200 import cm, harness  # noqa: E402
from paper_2507_13522_b200 import workloads as W  # noqa: E402

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
GPT2 = W.numels(W.gpt2_small())


def group(n, flags=0, place=cm.CM_SHADOW_HOST, dtype=cm.CM_F32, numel=GPT2):
    name = f"cmmb{os.getpid()}_{n}_{flags}_{place}"
    g = harness.VirtualGroup(numel, n, 0, dtype, W.CAP_BYTES, name, 2, place, flags)
    g._name = name
    return g


def close(g):
    g.sync()
    g.finalize()
    for r in range(g.n):
        cm.unlink_shadow(g._name, r)


def timed(g, fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    g.sync()
    for r in g.ranks:
        r.ctx.timing(True)
    for _ in range(iters):
        fn()
    g.sync()
    out = [r.ctx.timing(False) for r in g.ranks]
    return out


def adamw(impl=1):
    g = group(1, cm.CM_FLAG_NO_TAP)
    g.ranks[0].ctx.set_param("adamw_impl", impl)
    g.gen()
    def fn():
        g.allreduce()
        g.apply()
        g.t += 1
    (ms, cnt), = timed(g, fn, 20)
    P = g.ranks[0].padded
    avg = ms[1] / cnt[1]
    gbs = P * 28 / (avg * 1e-3) / 1e9
    close(g)
    return {"kernel": f"adamw_step fp32 impl={impl}", "elems": P, "avg_ms": avg, "hbm_GBps": gbs, "frac_of_measured": gbs / HBM}


def adamw_bf16(impl=1):
    g = group(1, cm.CM_FLAG_NO_TAP, dtype=cm.CM_BF16)
    g.ranks[0].ctx.set_param("adamw_impl", impl)
    g.gen()
    def fn():
        g.allreduce()
        g.apply()
        g.t += 1
    (ms, cnt), = timed(g, fn, 20)
    P = g.ranks[0].padded
    avg = ms[1] / cnt[1]
    gbs = P * 26 / (avg * 1e-3) / 1e9
    close(g)
    return {"kernel": f"adamw_step bf16 grads impl={impl}", "elems": P, "avg_ms": avg, "hbm_GBps": gbs, "frac_of_measured": gbs / HBM}


def gen():
    g = group(1, cm.CM_FLAG_NO_TAP)
    def fn():
        g.gen()
        g.t += 1
    (ms, cnt), = timed(g, fn, 20)
    P = g.ranks[0].padded
    avg = ms[3] / cnt[3]
    close(g)
    return {"kernel": "gen_grads fp32", "avg_ms": avg, "write_GBps": P * 4 / (avg * 1e-3) / 1e9}


def tap(flags=cm.CM_FLAG_TAP_DIRECT, label="rs_tap_ag n=1 (direct tap)", blocks=32):
    """All buckets of one iteration (kernel tap, or kernel + copy-engine tap), alone: the
    shadow runs only after the timed region."""
    g = group(1, flags)
    g.ranks[0].ctx.set_param("ar_blocks_tap_only", blocks)
    label += f" blocks={blocks}"
    g.gen()
    S = g.ranks[0].padded * 4
    tms = []
    for it in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(g.stream)
        g.allreduce()
        b.record(g.stream)
        g.apply()
        g.shadow()
        g.sync()
        g.t += 1
        if it >= 2:
            tms.append(a.elapsed_time(b))
    close(g)
    per_iter = sum(tms) / len(tms)
    return {"kernel": label, "ms_per_iter": per_iter, "tap_GBps": S / (per_iter * 1e-3) / 1e9}


def pcie():
    """Copy-engine pinned bandwidth: D2H alone, H2D alone, both at once (two streams)."""
    n = 512 << 20
    d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for name, ops in (("d2h", [(s1, lambda: h1.copy_(d1, non_blocking=True))]),
                      ("h2d", [(s1, lambda: d2.copy_(h2, non_blocking=True))]),
                      ("bidir", [(s1, lambda: h1.copy_(d1, non_blocking=True)),
                                 (s2, lambda: d2.copy_(h2, non_blocking=True))])):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(4):
            for st, f in ops:
                with torch.cuda.stream(st):
                    f()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out[name + "_GBps_each"] = 4 * n / dt / 1e9
    return {"kernel": "copy engines", **out}


def ar_virtual(n=8):
    """all ranks' buffers local: the reduce is HBM-bound (no NVLink); no tap."""
    g = group(n, cm.CM_FLAG_NO_TAP)
    g.gen()
    def fn():
        g.allreduce()
        g.apply()
        g.t += 1
    outs = timed(g, fn, 10)
    ms = sum(o[0][0] for o in outs) / 10
    S = g.ranks[0].padded * 4
    # per iteration all n launches read n*S/n... each rank reads n shards of S/n and writes n
    hbm = 2 * n * S / n * n / n
    close(g)
    return {"kernel": f"rs_ag virtual n={n} (HBM only)", "ms_per_iter_all_ranks": ms,
            "hbm_GBps": (2 * n * S) / (ms * 1e-3) / 1e9 / 1.0}


def shadow(place):
    g = group(1, 0, place)
    g.gen()
    def fn():
        g.allreduce()
        g.apply()
        g.shadow()
        g.t += 1
    (ms, cnt), = timed(g, fn, 10)
    L = g.ranks[0].ctx.info().shard_numel
    avg = ms[2] / cnt[2]
    h2d = L * 4
    d2h = L * (12 if place == cm.CM_SHADOW_HOST else 0)
    close(g)
    return {"kernel": f"shadow step ({'host' if place == 0 else 'device'} placement)", "avg_ms": avg,
            "h2d_GBps": h2d / (avg * 1e-3) / 1e9, "d2h_GBps": d2h / (avg * 1e-3) / 1e9,
            "step_ms_sum_of_classes": sum(ms[:4]) / 10}


TESTS = {"pcie": pcie, "adamw": adamw, "adamw_vec": lambda: adamw(0), "adamw_wt": lambda: adamw(2), "adamw_bf16": adamw_bf16,
         "adamw_bf16_vec": lambda: adamw_bf16(0), "adamw_bf16_wt": lambda: adamw_bf16(2),
         "adamw_wt1": lambda: adamw(3), "adamw_bf16_wt1": lambda: adamw_bf16(3), "gen": gen, "tap": tap,
         "tap16": lambda: tap(blocks=16), "tap64": lambda: tap(blocks=64), "tap148": lambda: tap(blocks=148),
         "tap_ce": lambda: tap(cm.CM_FLAG_TAP_COPYENGINE, "tap via copy engine (ablation)"),
         "tap_staged": lambda: tap(0, "staged tap (kernel -> HBM staging, copy-engine drain)"),
         "ar_virtual": ar_virtual, "shadow_host": lambda: shadow(cm.CM_SHADOW_HOST),
         "shadow_dev": lambda: shadow(cm.CM_SHADOW_DEVICE)}

if __name__ == "__main__":
    which = sys.argv[1:] or ["all"]
    if which == ["all"]:
        which = list(TESTS)
    for w in which:
        print(json.dumps({"test": w, **TESTS[w]()}), flush=True)
