"""Does host-bound DMA (the tap's device->host copies) slow the GPU's other work, and how?
One GPU.  Loads: none / D2H copies into pinned host memory (cudaHostAlloc, or an mmap'd
region registered with cudaHostRegister, optionally with transparent huge pages) running
back to back on a side stream.  Victims: (a) a bf16 GEMM loop (compute, few launches),
(b) a launch-bound loop of tiny kernels, (c) a GPT-2-like mix is covered by model mode.
Prints one JSON line per (load, victim)."""
import ctypes
import json
import mmap
import os
import sys
import time

import torch

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
libc = ctypes.CDLL("libc.so.6")
cudart = ctypes.CDLL("libcudart.so") if False else None


def thp_info():
    out = {}
    for f in ("enabled", "shmem_enabled", "defrag"):
        try:
            out[f] = open(f"/sys/kernel/mm/transparent_hugepage/{f}").read().strip()
        except OSError as e:
            out[f] = str(e)
    try:
        out["nr_hugepages"] = open("/proc/sys/vm/nr_hugepages").read().strip()
    except OSError as e:
        out["nr_hugepages"] = str(e)
    return out


def registered_host(nbytes, huge):
    """anonymous mmap (MADV_HUGEPAGE optionally), touched, registered with CUDA"""
    m = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    addr = ctypes.addressof(ctypes.c_char.from_buffer(m))
    if huge:
        libc.madvise(ctypes.c_void_p(addr), ctypes.c_size_t(nbytes), 14)   # MADV_HUGEPAGE
    ctypes.memset(addr, 0, nbytes)
    t = torch.frombuffer(m, dtype=torch.uint8)
    rc = torch.cuda.cudart().cudaHostRegister(t.data_ptr(), nbytes, 0)
    return t, m, rc


def run(victim, load, chunk_mb=32, seconds=3.0):
    nb = chunk_mb << 20
    src = torch.empty(nb, dtype=torch.uint8, device=dev)
    if load == "none":
        dst = None
    elif load == "pinned":
        dst = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    elif load in ("registered_4k", "registered_thp"):
        dst, keep, rc = registered_host(nb, load == "registered_thp")
    ls = torch.cuda.Stream(dev)
    a = torch.randn(8192, 4096, device=dev, dtype=torch.bfloat16)
    w = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
    o = torch.empty(8192, 4096, device=dev, dtype=torch.bfloat16)
    tiny = torch.zeros(1024, device=dev)

    def victim_step():
        if victim == "gemm":
            for _ in range(20):
                torch.mm(a, w, out=o)
        else:
            for _ in range(200):
                tiny.add_(1.0)

    # warm
    victim_step()
    torch.cuda.synchronize()
    n_load = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 0
    t_end = time.time() + seconds
    e0.record()
    while time.time() < t_end:
        if dst is not None and ls.query():
            with torch.cuda.stream(ls):
                for _ in range(8):
                    dst.copy_(src, non_blocking=True)
                    n_load += 1
        victim_step()
        reps += 1
        if reps % 10 == 0:
            torch.cuda.current_stream().synchronize()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    units = reps * (20 if victim == "gemm" else 200)
    return {"victim": victim, "load": load, "us_per_unit": ms * 1e3 / units,
            "load_GBps": n_load * nb / (ms * 1e-3) / 1e9, "reps": reps}


if __name__ == "__main__":
    print(json.dumps({"thp": thp_info()}), flush=True)
    for victim in ("gemm", "tiny"):
        for load in ("none", "pinned", "registered_4k", "registered_thp", "none"):
            try:
                print(json.dumps(run(victim, load)), flush=True)
            except Exception as e:  # noqa: BLE001
                print(json.dumps({"victim": victim, "load": load, "error": str(e)}), flush=True)
