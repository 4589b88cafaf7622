"""Host-to-device copy bandwidth of this box (pinned memory): one stream vs
two, chunk sizes, and the NUMA node of the pinned buffer (first touch under a
CPU affinity).  Diagnostics for the e2e leg (PCIe-bound)."""
import os
import time

import torch

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)


def bw(host, dst, streams, chunk, reps=3):
    n = host.numel()
    best = 0.0
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        i = 0
        k = 0
        while i < n:
            e = min(i + chunk, n)
            with torch.cuda.stream(streams[k % len(streams)]):
                dst[i:e].copy_(host[i:e], non_blocking=True)
            i = e
            k += 1
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        best = max(best, n / dt / 1e9)
    return best


N = 8 << 30
dst = torch.empty(N, dtype=torch.uint8, device=dev)
ncpu = os.cpu_count()
print("cpus", ncpu, "affinity", len(os.sched_getaffinity(0)))
try:
    nodes = sorted(d for d in os.listdir("/sys/devices/system/node") if d.startswith("node"))
    for nd in nodes:
        print(nd, open(f"/sys/devices/system/node/{nd}/cpulist").read().strip())
    print("gpu numa", open([p for p in [f"/sys/bus/pci/devices/{torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), 'pci_bus_id') else ''}/numa_node"] if os.path.exists(p)][0]).read().strip() if False else "")
except Exception as exc:
    print("numa info:", exc)
host = torch.empty(N, dtype=torch.uint8).pin_memory()
host.fill_(1)
s1 = [torch.cuda.Stream()]
s2 = [torch.cuda.Stream(), torch.cuda.Stream()]
for chunk in (64 << 20, 256 << 20, 1 << 30):
    print(f"chunk {chunk >> 20} MiB: 1 stream {bw(host, dst, s1, chunk):.1f} GB/s, 2 streams {bw(host, dst, s2, chunk):.1f} GB/s")
del host
allowed = sorted(os.sched_getaffinity(0))
half = len(allowed) // 2
for name, cpus in (("first half", allowed[:half]), ("second half", allowed[half:])):
    if not cpus:
        continue
    os.sched_setaffinity(0, set(cpus))
    h = torch.empty(N, dtype=torch.uint8).pin_memory()
    h.fill_(1)
    print(f"pinned under cpus {cpus[0]}-{cpus[-1]} ({name}): {bw(h, dst, s1, 256 << 20):.1f} GB/s")
    del h
os.sched_setaffinity(0, set(allowed))
