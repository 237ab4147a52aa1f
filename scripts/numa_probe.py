"""Does host NUMA placement explain e2e variance?  H2D bandwidth of a fresh pinned 2 GB buffer with the
process on (a) its default CPU set, (b) the GPU-local cores reported by NVML, (c) the other cores."""
import os, subprocess, time
import torch
import pynvml

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
local = {w * 64 + b for w, x in enumerate(words) for b in range(64) if (x >> b) & 1}
allc = set(os.sched_getaffinity(0))
print("cpus", len(allc), "gpu-local", len(local & allc))
print(subprocess.run("nvidia-smi topo -m; lscpu | grep -i numa", shell=True, capture_output=True, text=True).stdout)
n = 500_000_000
d = torch.empty(n, dtype=torch.int32, device="cuda")


def probe(tag, cpus):
    if cpus:
        os.sched_setaffinity(0, cpus)
    hb = torch.empty(n, dtype=torch.int32, pin_memory=True)
    hb.fill_(1)
    best = 0
    for _ in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        d.copy_(hb, non_blocking=True)
        torch.cuda.synchronize(); best = max(best, n * 4 / (time.perf_counter() - t) / 1e9)
    print(f"{tag}: H2D {best:.1f} GB/s")
    del hb


probe("default", None)
probe("gpu-local", local & allc)
other = allc - local
if other:
    probe("remote", other)
probe("gpu-local again", local & allc)
