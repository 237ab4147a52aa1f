"""H2D bandwidth probe: pinned 4 GB copy with torch and cudaMemcpyAsync chunks (diagnoses the e2e path)."""
import time, torch
n = 1_000_000_000
h = torch.empty(n, dtype=torch.int32, pin_memory=True)
d = torch.empty(n, dtype=torch.int32, device="cuda")
for chunk in (n, 64 << 20):
    torch.cuda.synchronize(); t = time.perf_counter()
    for i in range(0, n, chunk):
        d[i:i+chunk].copy_(h[i:i+chunk], non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"H2D chunk={chunk*4>>20} MB: {n*4/dt/1e9:.1f} GB/s")
torch.cuda.synchronize(); t = time.perf_counter()
h.copy_(d); torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"D2H {n*4/dt/1e9:.1f} GB/s")
print(torch.cuda.get_device_properties(0))
import subprocess; print(subprocess.run("nvidia-smi -q | grep -A8 -i 'PCI'", shell=True, capture_output=True, text=True).stdout[:3000])
