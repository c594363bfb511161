"""In-tree build of the engine library (nvcc, sm_100a only)."""

from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SOURCES = [os.path.join(HERE, "csrc", "tq_engine.cu"), os.path.join(HERE, "csrc", "tq_trunc.cu")]
HEADERS = [os.path.join(ROOT, "include", "tq_engine.h"), os.path.join(ROOT, "include", "tq_trunc.h"),
           os.path.join(HERE, "csrc", "tq_debug.cuh")]
LIB = os.path.join(HERE, "libtq_engine.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in SOURCES + HEADERS)


def build_library(force: bool = False, log_path: str | None = None) -> str:
    """Compile csrc/*.cu into libtq_engine.so (shared cudart so torch's runtime is reused)."""
    if not force and not needs_build():
        return LIB
    cmd = [nvcc_path(), "-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC", "-shared",
           "-cudart", "shared", "-Xptxas", "-v", "-diag-suppress", "177", "-o", LIB + ".tmp", *SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if log_path:
        with open(log_path, "w") as fh:
            fh.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stderr[-4000:])
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build_library(force=True, log_path=os.path.join(ROOT, "build_ptxas.log")))
