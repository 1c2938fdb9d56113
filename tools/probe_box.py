"""One-off probe of the GPU box: host cores, memory, topology, PCIe D2H/H2D bandwidth."""
import os, subprocess, time, json, torch
out = {}
out["cores_affinity"] = len(os.sched_getaffinity(0))
out["cpu_model"] = [l.split(":",1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
out["mem"] = open("/proc/meminfo").read().split("\n")[:3]
out["shm"] = subprocess.run("df -h /dev/shm", shell=True, capture_output=True, text=True).stdout
out["topo"] = subprocess.run("nvidia-smi topo -m", shell=True, capture_output=True, text=True).stdout
out["smi"] = subprocess.run("nvidia-smi --query-gpu=index,name,pci.bus_id,pcie.link.gen.max,pcie.link.width.max,clocks.max.sm --format=csv", shell=True, capture_output=True, text=True).stdout
out["numa"] = subprocess.run("lscpu | grep -i numa", shell=True, capture_output=True, text=True).stdout
n = 256 << 20
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
for name, fn in [("d2h", lambda: h.copy_(d, non_blocking=True)), ("h2d", lambda: d.copy_(h, non_blocking=True))]:
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); 
    for _ in range(10): fn()
    e.record(); torch.cuda.synchronize()
    out[name + "_GBps"] = 10 * n / (s.elapsed_time(e) * 1e-3) / 1e9
print(json.dumps(out, indent=1))
