"""C3: all-reduce bucket sweep, 1 MiB - 1 GiB, ours with tap / ours without tap / NCCL.

  python -m torch.distributed.run --nproc-per-node N tools/sweep_allreduce.py \
      --mode ours_tap|ours|nccl [--dtype f32|bf16] [--max-mib 1024] [--reps 20]
(NCCL without NVLS: run with NCCL_NVLS_ENABLE=0 in the environment.)

Per size: CUDA-event time of one all-reduce on the issuing stream (median of reps, max
over ranks), algBW = S/t, busBW = 2(n-1)/n * S/t (vs 770 GB/s measured peer / 900
nominal), tap GB/s per GPU = (S/n)/t.  Rank 0 prints one JSON line per size.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_13522_b200 import cm, harness  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="ours_tap", choices=["ours_tap", "ours_tap_direct", "ours", "nccl"])
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--min-mib", type=int, default=1)
    ap.add_argument("--max-mib", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--ar-blocks", type=int, default=0, help="grid cap override (0 = library default)")
    ap.add_argument("--min-kib", type=int, default=0, help="start size in KiB (overrides --min-mib)")
    ap.add_argument("--max-kib", type=int, default=0, help="end size in KiB (overrides --max-mib)")
    ap.add_argument("--nvls", action="store_true", help="CM_FLAG_NVLS: one-shot push via multimem.st")
    ap.add_argument("--tag", default="", help="free-form label copied into every output line")
    ap.add_argument("--multi-bucket", action="store_true",
                    help="ours: the burst is `burst` DIFFERENT buckets of one iteration (as in a training step: "
                         "the next bucket's kernel may launch early, PDL) instead of one bucket over iterations")
    ap.add_argument("--burst", type=int, default=1,
                    help="launches per timed rep (back to back, as in a step); time = total / burst")
    ap.add_argument("--oneshot-max", type=int, default=-1,
                    help="one-shot push kernel for buckets <= this many bytes (-1 = library default, 0 = off)")
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, rank = dist.get_world_size(), dist.get_rank()
    dtype = cm.CM_F32 if args.dtype == "f32" else cm.CM_BF16
    es = 4 if dtype == cm.CM_F32 else 2
    dev = torch.device("cuda", local)
    kib = args.min_kib or args.min_mib * 1024
    kib_max = args.max_kib or args.max_mib * 1024
    while kib <= kib_max:
        S = kib << 10
        mib = kib
        numel = [S // es] * (args.burst if args.multi_bucket and args.mode != "nccl" else 1)
        stream = torch.cuda.Stream(dev, priority=-1)
        if args.mode == "nccl":
            buf = torch.randn(S // es, device=dev).to(harness.TORCH_DT[dtype])
            fn = lambda t: dist.all_reduce(buf)   # noqa: E731
            ctx = None
        else:
            flags = {"ours_tap": cm.CM_FLAG_NO_SHADOW, "ours": cm.CM_FLAG_NO_TAP,
                     "ours_tap_direct": cm.CM_FLAG_NO_SHADOW | cm.CM_FLAG_TAP_DIRECT}[args.mode]
            name = f"cmsw_{os.environ.get('MASTER_PORT', '0')}_{mib}"
            if args.nvls:
                flags |= cm.CM_FLAG_NVLS
            R = harness.DistRank(numel, dtype, S, name, 2, cm.CM_SHADOW_HOST, flags)
            if args.ar_blocks:
                R.r.ctx.set_param("ar_blocks", args.ar_blocks)
            # each launch is timed as a complete collective (exit barrier on); in a training
            # step the exits are lazy and the optimizer's entry barrier fences the iteration
            R.r.ctx.set_param("lazy_exit", int(os.environ.get("CM_LAZY_EXIT_SWEEP", "0")))
            if args.oneshot_max >= 0:
                R.r.ctx.set_param("oneshot_max_bytes", args.oneshot_max)
            R.r.ctx.gen_grads(0, 0, 10, R.stream)
            R.stream.synchronize()
            stream = R.stream
            ctx = R.r.ctx
            if args.multi_bucket:
                nbk = R.n_buckets
                fn = lambda t: ctx.allreduce_multicast(t % nbk, t // nbk, stream)   # noqa: E731
            else:
                fn = lambda t: ctx.allreduce_multicast(0, t, stream)   # noqa: E731
        times = []
        it = 0
        with torch.cuda.stream(stream):
            for t in range(args.warmup + args.reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                for _ in range(args.burst):
                    fn(it)
                    it += 1
                b.record(stream)
                b.synchronize()
                if t >= args.warmup:
                    times.append(a.elapsed_time(b) / args.burst)
        med = statistics.median(times)
        tt = torch.tensor([med], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        med = tt.item()
        if rank == 0:
            sec = med * 1e-3
            print(json.dumps({"tag": args.tag, "multi_bucket": args.multi_bucket, "mode": args.mode + ("_nvls" if args.nvls else ""), "burst": args.burst, "ar_blocks": args.ar_blocks, "oneshot_max": args.oneshot_max, "nvls": os.environ.get("NCCL_NVLS_ENABLE", "default"),
                              "dtype": args.dtype, "n": n, "bytes": S, "ms": med,
                              "p10_ms": sorted(times)[len(times) // 10], "p90_ms": sorted(times)[9 * len(times) // 10],
                              "algbw_GBps": S / sec / 1e9, "busbw_GBps": 2 * (n - 1) / n * S / sec / 1e9,
                              "tap_GBps_per_gpu": (S / n) / sec / 1e9 if args.mode.startswith("ours_tap") else 0.0}),
                  flush=True)
        if ctx is not None:
            dist.barrier()
            ctx.finalize()
            cm.unlink_shadow(name, rank)
        dist.barrier()
        kib *= 2
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
