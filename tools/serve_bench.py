"""Shadow serving throughput at GPT-2 size: n virtual ranks on one GPU train
a few steps with host snapshots every K; then, from the host segments alone, time
- the consolidated fetch of p, m, v (1.49 GB) with 1, 4 and 8 reader threads,
- one tensor (the 38.6 M-element wte) from the shards that own it,
- the per-tensor model file export (cm_shadow_export) to /dev/shm,
and a fetch while the group keeps training.  Prints one JSON line.

  python tools/serve_bench.py [--n 2] [--steps 4]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2507_13522_b200 import cm, harness, serving  # noqa: E402
from paper_2507_13522_b200 import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2)
    ap.add_argument("--steps", type=int, default=4)
    args = ap.parse_args()
    numel = W.numels(W.gpt2_small())
    name = f"cmsrvb{os.getpid()}"
    g = harness.VirtualGroup(numel, args.n, 0, cm.CM_F32, W.CAP_BYTES, name, 3, cm.CM_SHADOW_HOST, 0,
                             persist_every=2)
    smap = serving.ShardMap(numel, cm.CM_F32, W.CAP_BYTES, args.n)
    out = {"tool": "serve_bench", "n_virtual_ranks": args.n, "params": sum(numel), "padded": smap.padded}
    try:
        for _ in range(args.steps):
            g.step()
        g.sync()
        I = serving.consolidate(name, args.n)
        out["consolidated_step"] = I
        nbytes = 3 * 4 * smap.padded
        for th in (1, 4, 8):
            best = 1e9
            for _ in range(3):
                t0 = time.perf_counter()
                serving.fetch(name, smap, threads=th, verify=False)
                best = min(best, time.perf_counter() - t0)
            out[f"fetch_pmv_GBps_threads{th}"] = nbytes / best / 1e9
        t0 = time.perf_counter()
        serving.fetch(name, smap, threads=8, verify=True)
        out["fetch_pmv_GBps_threads8_crc_checked"] = nbytes / (time.perf_counter() - t0) / 1e9
        wte = max(range(len(numel)), key=lambda i: numel[i])
        t0 = time.perf_counter()
        serving.fetch_tensor(name, smap, wte, what="p")
        out["fetch_wte_p_ms"] = (time.perf_counter() - t0) * 1e3
        path = f"/dev/shm/{name}.model"
        t0 = time.perf_counter()
        serving.export(name, numel, cm.CM_F32, W.CAP_BYTES, args.n, path)
        out["export_s"] = time.perf_counter() - t0
        out["export_bytes"] = os.path.getsize(path)
        os.unlink(path)
        # while training: issue steps without waiting, fetch, count refusals
        ok = refused = 0
        for _ in range(4):
            g.step()
            g.step()
            try:
                serving.fetch(name, smap, what=("p",), threads=8)
                ok += 1
            except cm.CMError as e:
                assert e.status == cm.CM_ERR_STATE
                refused += 1
        g.sync()
        out["fetch_during_training"] = {"ok": ok, "refused_torn_or_rewritten": refused}
    finally:
        g.sync()
        g.finalize()
        for r in range(args.n):
            cm.unlink_shadow(name, r)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
