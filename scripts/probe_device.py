"""Print the device/host facts the design depends on (L2 size, persisting limits, SM count, host cores)."""
import os, json, subprocess
import torch
p = torch.cuda.get_device_properties(0)
out = {"name": p.name, "sms": p.multi_processor_count, "l2": getattr(p, "L2_cache_size", None),
       "mem": p.total_memory, "cc": [p.major, p.minor], "host_cores": os.cpu_count()}
try:
    from cuda.bindings import runtime as rt
    for a in ["cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrMaxAccessPolicyWindowSize", "cudaDevAttrL2CacheSize",
              "cudaDevAttrMaxSharedMemoryPerBlockOptin", "cudaDevAttrMaxRegistersPerMultiprocessor", "cudaDevAttrClockRate", "cudaDevAttrMemoryClockRate", "cudaDevAttrGlobalMemoryBusWidth"]:
        err, v = rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, a), 0)
        out[a] = v
except Exception as e:
    out["cuda_python_err"] = repr(e)
print(json.dumps(out, indent=1))
print(subprocess.run("lscpu | head -20; nvidia-smi; free -g", shell=True, capture_output=True, text=True).stdout)
