"""NVLink hardware counters around the lockstep all-reduce chain (and ZeRO-1's reduce-scatter +
parameter all-gather): per-GPU bytes transmitted / received over all NVLink links, read with
NVML field counters before and after K iterations, against the algorithmic bytes and the
event-timed chain duration.  One process per GPU:

  python -m torch.distributed.run --nproc-per-node N tools/nvlink_counters.py [--steps 20] [--zero1]
Rank 0 prints one JSON line (every rank's counters gathered)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_13522_b200 import cm, harness  # noqa: E402
from paper_2507_13522_b200 import workloads as W  # noqa: E402

FIELDS = {"xmit_bytes": 202, "rcv_bytes": 204, "tput_tx_kib": 138, "tput_rx_kib": 139}


def counters(index):
    import pynvml as N
    N.nvmlInit()
    h = N.nvmlDeviceGetHandleByIndex(index)
    out = {}
    for name, fid in FIELDS.items():
        tot, ok = 0, 0
        for link in range(18):
            try:
                v = N.nvmlDeviceGetFieldValues(h, [(fid, link)])[0]
                if v.nvmlReturn == 0:
                    tot += int(v.value.ullVal)
                    ok += 1
            except Exception:   # noqa: BLE001 -- field not supported on this driver / link
                pass
        out[name] = tot if ok else None
        out[name + "_links"] = ok
    N.nvmlShutdown()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--zero1", action="store_true")
    a = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, rank = dist.get_world_size(), dist.get_rank()
    numel = W.numels(W.gpt2_small())
    flags = cm.CM_FLAG_NO_TAP | (cm.CM_FLAG_ZERO1 if a.zero1 else 0)
    R = harness.DistRank(numel, cm.CM_F32, W.CAP_BYTES, "unused", 2, cm.CM_SHADOW_HOST, flags)
    c = R.r.ctx
    info = c.info()
    S = info.padded_numel * 4
    for _ in range(3):
        R.step()
    R.sync()
    dist.barrier()
    torch.cuda.synchronize()
    before = counters(local)
    ev = []
    for _ in range(a.steps):
        c.gen_grads(R.seed, R.t, R.gscale, R.stream)
        c.barrier(R.stream)
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(R.stream)
        for b in range(R.n_buckets):
            c.allreduce_multicast(b, R.t, R.stream)
        e1.record(R.stream)
        c.apply_step(R.t + 1, stream=R.stream, **R.hp)
        e2.record(R.stream)
        R.t += 1
        ev.append((e0, e1, e2))
    R.sync()
    torch.cuda.synchronize()
    after = counters(local)
    chain_ms = sum(x.elapsed_time(y) for x, y, _ in ev) / a.steps
    opt_ms = sum(y.elapsed_time(z) for _, y, z in ev) / a.steps
    mine = {"rank": rank, "chain_ms": chain_ms, "opt_ms": opt_ms,
            "delta": {k: (after[k] - before[k]) if after.get(k) is not None and before.get(k) is not None else None
                      for k in FIELDS}, "links": {k: after[k + "_links"] for k in FIELDS}}
    allr = [None] * n
    dist.all_gather_object(allr, mine)
    if rank == 0:
        if a.zero1:   # reduce-scatter: (n-1)/n S each way; parameter all-gather: (n-1)/n 4P each way
            algo = (n - 1) / n * S + (n - 1) / n * info.padded_numel * 4
        else:         # two-shot: reduce-scatter + all-gather, 2 (n-1)/n S each way
            algo = 2 * (n - 1) / n * S
        for r in allr:
            d = r["delta"]
            per_it = {k: (v / a.steps if v is not None else None) for k, v in d.items()}
            r["per_iteration_bytes"] = per_it
            x = per_it.get("xmit_bytes")
            if x:
                r["tx_over_algorithmic"] = x / algo
                r["rx_over_algorithmic"] = per_it["rcv_bytes"] / algo if per_it.get("rcv_bytes") else None
                t_s = (r["chain_ms"] + (r["opt_ms"] if a.zero1 else 0.0)) * 1e-3
                r["tx_GBps_over_window"] = x / t_s / 1e9
        print(json.dumps({"n": n, "zero1": a.zero1, "steps": a.steps, "S_bytes": S,
                          "algorithmic_bytes_per_iteration_per_direction": algo, "ranks": allr,
                          "what": "NVML NVLink byte counters (fields 202/204: tx/rx bytes per link, summed over "
                                  "links; 138/139: data throughput counters in KiB) around K iterations of the "
                                  "lockstep step; window = the all-reduce chain (+ the ZeRO-1 optimizer)"}),
              flush=True)
    dist.barrier()
    c.finalize()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
