"""Build the sm_100a shared libraries in-tree (no JIT cache; the .so files travel
to the GPU box with the repo snapshot).

  lib/libocclb200.so : the product -- daemon kernel + host runtime behind include/occl.h
  lib/libocclgen.so  : test/bench support -- the seeded input generator on the GPU
  lib/libocclbench.so: bench support -- native per-rank latency harness over the C-ABI
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "lib")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
                 "-I" + os.path.join(ROOT, "include"), "-Xptxas", "-v", "-maxrregcount=104", "-lpthread"]

TARGETS = {
    "libocclb200.so": ["occl_daemon.cu", "occl_host.cc"],
    "libocclgen.so": ["testgen.cu"],
    "libocclbench.so": ["bench_native.cc"],     # bench / test harness over the C-ABI (links the product)
}
LINK = {"libocclbench.so": ["-L" + LIB, "-locclb200", "-Xlinker", "-rpath=$ORIGIN"]}


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = [os.path.join(CSRC, s) for s in srcs] + [os.path.join(CSRC, "occl_internal.h"),
                                                     os.path.join(ROOT, "include", "occl.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> list[str]:
    os.makedirs(LIB, exist_ok=True)
    built = []
    for name, srcs in TARGETS.items():
        out = os.path.join(LIB, name)
        if not force and not _stale(out, srcs):
            continue
        cmd = [NVCC] + COMMON + [os.path.join(CSRC, s) for s in srcs] + LINK.get(name, []) + ["-o", out + ".tmp"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed building {name}")
        if verbose:
            sys.stderr.write(r.stderr)
        os.replace(out + ".tmp", out)
        built.append(out)
    return built


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
