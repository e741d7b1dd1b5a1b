"""Compile the oracle's C restatements (TEST INFRASTRUCTURE) with gcc:

    python oracle/build_oracle.py         # or __graft_entry__.build()

oracle/precond_oracle.c -> oracle/libprecond_oracle.so (git-ignored like every
built object; it travels to the GPU box with the repo snapshot).  -O2 without
floating-point contraction, so every product and sum rounds once, as in the
reference's numba code.
"""

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "precond_oracle.c")
OUT = os.path.join(HERE, "libprecond_oracle.so")


def build(force=False, quiet=True):
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= os.path.getmtime(SRC):
        return OUT
    gcc = shutil.which("gcc") or "gcc"
    cmd = [gcc, "-O2", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC", "-o", OUT, SRC, "-lm"]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("gcc failed for the oracle:\n" + out.stderr[-2000:])
    if not quiet:
        print(f"built {OUT}")
    return OUT


if __name__ == "__main__":
    build(force=True, quiet=False)
