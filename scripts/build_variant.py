#!/usr/bin/env python
"""Build the product library (and the native bench harness linked to it) from the
csrc/ of another git revision, or with extra -D defines, into a separate
directory -- for interleaved A/B runs on one lease (OCCL_LIB_PATH=<dir>/libocclb200.so).

  python scripts/build_variant.py --out paper_2303_06324_b200/lib_ab/base --rev HEAD~1
  python scripts/build_variant.py --out paper_2303_06324_b200/lib_ab/x -D OCCL_SOMETHING=1
"""
import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2303_06324_b200 import build as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--rev", default="")
    ap.add_argument("-D", action="append", default=[])
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    tmp = tempfile.mkdtemp()
    csrc = B.CSRC
    inc = os.path.join(ROOT, "include")
    if a.rev:
        for sub in ("paper_2303_06324_b200/csrc", "include"):
            os.makedirs(os.path.join(tmp, sub), exist_ok=True)
            files = subprocess.run(["git", "ls-tree", "--name-only", a.rev, sub + "/"], cwd=ROOT, capture_output=True,
                                   text=True, check=True).stdout.split()
            for f in files:
                data = subprocess.run(["git", "show", f"{a.rev}:{f}"], cwd=ROOT, capture_output=True, check=True).stdout
                with open(os.path.join(tmp, f), "wb") as fh:
                    fh.write(data)
        csrc = os.path.join(tmp, "paper_2303_06324_b200/csrc")
        inc = os.path.join(tmp, "include")
    common = [x for x in B.COMMON if not x.startswith("-I")] + ["-I" + inc] + ["-D" + d for d in a.D]
    for name in ("libocclb200.so", "libocclbench.so"):
        srcs = [os.path.join(csrc, s) for s in B.TARGETS[name]]
        link = ["-L" + a.out, "-locclb200", "-Xlinker", "-rpath=$ORIGIN"] if name == "libocclbench.so" else []
        cmd = [B.NVCC] + common + srcs + link + ["-o", os.path.join(a.out, name)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.stderr.write(r.stderr)
            sys.exit(1)
    shutil.rmtree(tmp)
    print(a.out)


if __name__ == "__main__":
    main()
