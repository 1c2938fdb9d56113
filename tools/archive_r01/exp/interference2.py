"""Victim slowdown vs device->host traffic intensity (one GPU): copy engine at full speed vs
a one-CTA SM trickle at a target rate.  Harm is reported per GB moved."""
import ctypes
import json
import os
import time

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
L = ctypes.CDLL(os.path.join(HERE, "libtrickle.so"))
L.launch_trickle.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_int,
                             ctypes.c_void_p]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
NB = 64 << 20
src = torch.empty(NB, dtype=torch.uint8, device=dev)
dst = torch.empty(NB, dtype=torch.uint8, pin_memory=True)
ls = torch.cuda.Stream(dev, priority=0)
tiny = torch.zeros(1024, device=dev)
a = torch.randn(8192, 4096, device=dev, dtype=torch.bfloat16)
w = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
o = torch.empty(8192, 4096, device=dev, dtype=torch.bfloat16)


def victim(kind):
    if kind == "tiny":
        for _ in range(200):
            tiny.add_(1.0)
        return 200
    for _ in range(4):
        torch.mm(a, w, out=o)
    return 4


def run(kind, load, gap_ns=0, seconds=3.0):
    victim(kind)
    torch.cuda.synchronize()
    moved = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    units = 0
    it = 0
    t_end = time.time() + seconds
    e0.record()
    while time.time() < t_end:
        if load != "none" and ls.query():
            if load == "ce":
                with torch.cuda.stream(ls):
                    dst.copy_(src, non_blocking=True)
            else:
                L.launch_trickle(src.data_ptr(), dst.data_ptr(), NB, gap_ns, 16384, ls.cuda_stream)
            moved += NB
        units += victim(kind)
        it += 1
        if it % 20 == 0:
            torch.cuda.current_stream().synchronize()
    e1.record()
    torch.cuda.synchronize()
    ls.synchronize()
    ms = e0.elapsed_time(e1)
    return {"victim": kind, "load": load, "gap_ns": gap_ns, "us_per_unit": ms * 1e3 / units,
            "load_GBps": moved / (ms * 1e-3) / 1e9, "ms": ms}


base = {}
for kind in ("tiny", "gemm"):
    r = run(kind, "none")
    base[kind] = r["us_per_unit"]
    print(json.dumps(r), flush=True)
    for load, gap in (("ce", 0), ("sm", 0), ("sm", 1000), ("sm", 3000), ("sm", 8000), ("sm", 20000)):
        r = run(kind, load, gap)
        slow = r["us_per_unit"] / base[kind] - 1
        r["slowdown"] = slow
        r["harm_pct_per_GBps"] = 100 * slow / max(r["load_GBps"], 1e-9)
        print(json.dumps(r), flush=True)
