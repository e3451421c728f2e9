"""Build ``libges_b200.so`` in-tree with nvcc for sm_100a (no JIT cache)."""

from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SOURCES = ("ges_abi.cu", "ges_prep.cu", "ges_bin.cu", "ges_tile.cu", "ges_train.cu", "ges_f64.cu")
OUT = os.path.join(HERE, "libges_b200.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-cudart", "static"]


def _nvcc():
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "ges_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = OUT, extra=()) -> str:
    if not force and out == OUT and not stale():
        return OUT
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-o", out + ".tmp", *[os.path.join(CSRC, s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    import sys
    if len(sys.argv) > 1 and sys.argv[1] == "stats":   # tuning build with work counters
        print(build(force=True, verbose=True, out=os.path.join(HERE, "libges_b200_stats.so"),
                    extra=("-DGES_STATS",)))
    else:
        print(build(force=True, verbose=True))
