"""Build the in-tree CUDA libraries for sm_100a with nvcc (no torch JIT, no site-packages install).

    libara.so        the product: C ABI of include/ara.h (csrc/*.cu)
    libara_synth.so  the seeded device input generator (synth/synth.cu; test/bench infrastructure)
    libara_testing.so  test-only read-back of a context's tables (csrc/testing.cu, include/ara_testing.h)
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
INCLUDE = os.path.join(ROOT, "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I", INCLUDE, "-Xptxas", "-warn-spills"]

LIBS = {
    "libara.so": [os.path.join(HERE, "csrc", f) for f in ("ara_api.cu", "metrics.cu", "kernels_presence.cu", "kernels_presence_mid.cu", "kernels_presence_wide.cu", "kernels_dense.cu", "kernels_study.cu", "outputs.cu", "kernels_stream.cu")],
    "libara_synth.so": [os.path.join(HERE, "synth", "synth.cu")],
    "libara_testing.so": [os.path.join(HERE, "csrc", "testing.cu")],
}
DEPS = {
    # every header under csrc/ (a kernel header missing here once left a stale libara.so in place)
    "libara.so": sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [os.path.join(INCLUDE, "ara.h")],
    "libara_synth.so": [os.path.join(INCLUDE, "ara_synth.h")],
    "libara_testing.so": sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [os.path.join(INCLUDE, "ara.h"),
                                                                                 os.path.join(INCLUDE, "ara_testing.h")],
}
OUT_DIR = {"libara.so": HERE, "libara_synth.so": os.path.join(HERE, "synth"), "libara_testing.so": HERE}


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def _compile(src, obj, verbose):
    cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def build(force: bool = False, verbose: bool = False) -> None:
    for lib, srcs in LIBS.items():
        out = os.path.join(OUT_DIR[lib], lib)
        if not force and not _stale(out, srcs + DEPS[lib]):
            continue
        objdir = os.path.join(ROOT, "build", "obj")
        os.makedirs(objdir, exist_ok=True)
        objs = [os.path.join(objdir, os.path.basename(s) + ".o") for s in srcs]
        with ThreadPoolExecutor(max_workers=len(srcs)) as ex:
            list(ex.map(lambda so: _compile(so[0], so[1], verbose), zip(srcs, objs)))
        # static cudart (nvcc default): no dependency on which libcudart torch loaded
        cmd = [NVCC, *ARCH, "-shared", "-o", out, *objs, "-cudart", "static"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
