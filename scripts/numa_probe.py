"""Pinned-host H2D bandwidth vs the NUMA node the pinned pages were allocated
from (CPU affinity of the allocating thread), to explain the C5 variance."""
import os, glob, torch
nodes = sorted(glob.glob("/sys/devices/system/node/node[0-9]*"))
def cpus(n):
    out = []
    for part in open(f"{n}/cpulist").read().strip().split(","):
        a, _, b = part.partition("-")
        out += list(range(int(a), int(b or a) + 1))
    return out
print("nodes:", [(os.path.basename(n), len(cpus(n))) for n in nodes])
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    print("gpu numa node (nvml):", getattr(pynvml, "nvmlDeviceGetNumaNodeId", lambda h: "n/a")(h))
except Exception as e:
    print("nvml:", e)
dev = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
full = os.sched_getaffinity(0)
for n in nodes:
    c = set(cpus(n)) & full
    if not c:
        continue
    os.sched_setaffinity(0, c)
    for rep in range(2):
        h = torch.empty(2 << 30, dtype=torch.uint8, pin_memory=True)
        h.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dev.copy_(h, non_blocking=True)
        a.record(); 
        for _ in range(3): dev.copy_(h, non_blocking=True)
        b.record(); torch.cuda.synchronize()
        print(os.path.basename(n), "rep", rep, "H2D %.1f GB/s" % (3 * (2 << 30) / a.elapsed_time(b) / 1e6))
        del h
os.sched_setaffinity(0, full)
