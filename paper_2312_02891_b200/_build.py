"""Build libsylvadi_b200.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2312_02891_b200._build [--force]
"""

import glob
import os
import shutil
import subprocess
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC_DIR = os.path.join(_HERE, "csrc")
SOURCES = [os.path.join(SRC_DIR, "sad_capi.cu")]
DEPS = SOURCES + sorted(glob.glob(os.path.join(SRC_DIR, "*.cuh"))) + [
    os.path.join(os.path.dirname(_HERE), "include", "sylvadi_b200.h")]
OUT = os.path.join(_HERE, "libsylvadi_b200.so")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
              "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def nvcc():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date():
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force=False, verbose=False):
    if not force and up_to_date():
        return OUT
    cmd = [nvcc()] + NVCC_FLAGS + ["-o", OUT] + SOURCES
    log_path = os.path.join(_HERE, "csrc", "build.log")
    proc = subprocess.run(cmd, capture_output=True, text=True)
    with open(log_path, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + proc.stdout + proc.stderr)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed ({proc.returncode}); see {log_path}\n"
                           + proc.stderr[-4000:])
    if verbose:
        print(f"built {OUT}")
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
