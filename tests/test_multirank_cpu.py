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


def test_bench_reference_arm_under_torchrun_world2():
    """--impl reference under torchrun: rank 0 alone prints one JSON line, others exit 0."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nproc-per-node=2", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", "bench.py", "--impl", "reference", "--gpus", "2",
           "--workload", "c1", "--cpu-sample-s", "0.3"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0
