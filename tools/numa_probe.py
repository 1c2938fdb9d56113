"""Host-link probe: does the NUMA node of the pinned host buffer matter for D2H?

Launch with torchrun (one rank per GPU).  Each rank maps an anonymous shared region,
binds it (mbind, MPOL_BIND) to NUMA node `k`, pins it (cudaHostRegister) and times
copy-engine D2H copies into it: alone (rank by rank) and all ranks at once, for k = the
GPU's own node and every other node.  Prints one JSON line per (mode, node policy)."""
import ctypes
import json
import mmap
import os
import time

import numpy as np
import torch
import torch.distributed as dist

SYS_mbind = 237          # x86_64
MPOL_BIND = 2
libc = ctypes.CDLL("libc.so.6", use_errno=True)


def gpu_node(dev):
    p = torch.cuda.get_device_properties(dev)
    bus = "%04x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
    path = f"/sys/bus/pci/devices/{bus.lower()}/numa_node"
    try:
        return int(open(path).read().strip()), bus
    except OSError:
        return -1, bus


def nodes():
    base = "/sys/devices/system/node"
    return sorted(int(d[4:]) for d in os.listdir(base) if d.startswith("node") and d[4:].isdigit())


def bound_pinned(nbytes, node):
    libc.mmap.restype = ctypes.c_void_p
    libc.mmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long]
    addr = libc.mmap(None, nbytes, mmap.PROT_READ | mmap.PROT_WRITE, mmap.MAP_SHARED | mmap.MAP_ANONYMOUS, -1, 0)
    if node >= 0:
        mask = ctypes.c_ulong(1 << node)
        rc = libc.syscall(SYS_mbind, ctypes.c_void_p(addr), ctypes.c_ulong(nbytes), MPOL_BIND,
                          ctypes.byref(mask), ctypes.c_ulong(64), 0)
        if rc != 0:
            raise OSError(ctypes.get_errno(), "mbind")
    rt = torch.cuda.cudart()
    r = rt.cudaHostRegister(addr, nbytes, 0)
    assert int(r) == 0, r
    t = torch.from_numpy(np.ctypeslib.as_array((ctypes.c_uint8 * nbytes).from_address(addr)))
    return addr, t


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    my_node, bus = gpu_node(local)
    allnodes = nodes()
    info = dict(rank=rank, bus=bus, node=my_node, nodes=allnodes, cpus=len(os.sched_getaffinity(0)))
    infos = [None] * world
    dist.all_gather_object(infos, info)
    if rank == 0:
        print(json.dumps({"topology": infos}), flush=True)
    nbytes = 512 << 20
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d.fill_(1)
    pols = [("local", my_node)] + [(f"node{k}", k) for k in allnodes if k != my_node] + [("default", -1)]
    # every rank must run the same number of policies
    npol = [None] * world
    dist.all_gather_object(npol, len(pols))
    pols = pols[: min(npol)]
    for name, node in pols:
        addr, h = bound_pinned(nbytes, node)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3):
            h.copy_(d, non_blocking=True)
        torch.cuda.synchronize()
        res = {}
        for mode in ("alone", "concurrent"):
            times = []
            for who in (range(world) if mode == "alone" else [None]):
                dist.barrier()
                if who is None or who == rank:
                    s.record()
                    for _ in range(8):
                        h.copy_(d, non_blocking=True)
                    e.record()
                    torch.cuda.synchronize()
                    times.append(s.elapsed_time(e) * 1e-3)
                dist.barrier()
            gbps = 8 * nbytes / max(times) / 1e9
            allv = [None] * world
            dist.all_gather_object(allv, gbps)
            res[mode] = allv
        if rank == 0:
            print(json.dumps({"policy": name, "note": "rank 0's node choice; other ranks use their own 'local'/'nodeK' in the same position",
                              "d2h_GBps_alone": res["alone"], "d2h_GBps_concurrent": res["concurrent"]}), flush=True)
        torch.cuda.cudart().cudaHostUnregister(addr)
        del h
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
