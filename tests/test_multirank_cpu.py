"""World-size-2 host-logic tests on CPU (gloo): the bench's launch/rank-0-prints contract,
max-over-ranks timing, and the blob exchange used by cm_connect."""
import json
import os
import socket
import subprocess
import sys

import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    import bench
    m = bench.max_over_ranks(10.0 + rank)
    blobs = [None] * world
    dist.all_gather_object(blobs, bytes([rank]) * 16)        # the cm_connect blob exchange
    q.put((rank, m, blobs))
    dist.destroy_process_group()


def test_max_over_ranks_and_blob_exchange_gloo():
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(60)
    for rank, m, blobs in out:
        assert m == 11.0
        assert blobs == [bytes([0]) * 16, bytes([1]) * 16]


def _partition_worker(rank, world, port, q):
    """Each rank derives its shards from the library's plan (host-only ABI) and every
    rank's element ranges are exchanged over gloo, as the blobs are."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    from paper_2507_13522_b200 import cm
    from paper_2507_13522_b200 import workloads as W
    out = {}
    for name, numel, dt in (("gpt2", W.numels(W.gpt2_small()), cm.CM_F32),
                            ("ragged_bf16", W.numels(W.c1_ragged()) + [5, 3, 70001], cm.CM_BF16)):
        table = cm.plan_bucket_table(numel, dt, 1 << 20 if name != "gpt2" else W.CAP_BYTES, world)
        mine = [(off + rank * (pad // world), off + (rank + 1) * (pad // world)) for off, pad, _ in table]
        allr = [None] * world
        dist.all_gather_object(allr, mine)
        out[name] = (table, allr, cm.plan_buckets(numel, dt, 1 << 20 if name != "gpt2" else W.CAP_BYTES, world)[0])
    q.put((rank, out))
    dist.destroy_process_group()


def test_rank_to_shard_partition_gloo():
    """contiguous shard r of every bucket -> rank r.  Over world size 2 the ranks'
    shards are 16-byte aligned, equal per bucket, disjoint, and cover every padded element
    exactly once; the real elements are all covered."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_partition_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(60)
    for name in res[0][1]:
        table, allr, total = res[0][1][name]
        assert res[1][1][name][1] == allr                 # both ranks agree on the partition
        es = 4 if name == "gpt2" else 2
        cover = []
        for r, ranges in enumerate(allr):
            for (lo, hi), (off, pad, used) in zip(ranges, table):
                assert (hi - lo) * 2 == pad and (lo * es) % 16 == 0 and ((hi - lo) * es) % 16 == 0
                cover.append((lo, hi))
        cover.sort()
        assert cover[0][0] == 0 and cover[-1][1] == total
        assert all(a[1] == b[0] for a, b in zip(cover, cover[1:]))   # disjoint, no gap
        assert sum(u for _, _, u in table) <= total


def test_bench_reference_arm_under_torchrun_world2():
    """--impl reference under torchrun: rank 0 alone prints one JSON line, others exit 0."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nproc-per-node=2", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", "bench.py", "--impl", "reference", "--gpus", "2",
           "--workload", "c1", "--steps", "2", "--warmup", "1"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0
    assert d["steps"] == 2 and d["warmup"] == 1 and d["cpu_baseline"]["steps"] == 2
