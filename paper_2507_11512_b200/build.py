"""Build libhpgmxp.so in-tree for sm_100a (nvcc; no torch extension machinery).

    python -m paper_2507_11512_b200.build
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libhpgmxp.so")

NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def sources():
    return sorted(os.path.join(SRC, f) for f in os.listdir(SRC) if f.endswith(".cu"))


def deps():
    return sources() + sorted(os.path.join(SRC, f) for f in os.listdir(SRC)
                              if f.endswith((".h", ".cuh"))) + [os.path.join(ROOT, "include", "hpgmxp.h")]


def up_to_date():
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in deps())


def build(force=False, verbose=False):
    if not force and up_to_date():
        return OUT
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-I", SRC, *sources(),
           "-o", OUT + ".tmp", "-lnccl"]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        sys.stderr.write(p.stdout + p.stderr)
        raise RuntimeError("nvcc failed building libhpgmxp.so")
    if verbose:
        sys.stderr.write(p.stderr)
    os.replace(OUT + ".tmp", OUT)
    with open(os.path.join(HERE, "ptxas_info.txt"), "w") as f:
        f.write(p.stderr)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
