"""Install the reference package `sylvadi` into oracle/_ref/ (TEST INFRASTRUCTURE).

The reference (/root/reference/pkg, pure Python + numba) is installed, unmodified,
with pip from a copy under /tmp (the reference tree is read-only), without
dependency resolution (numpy / scipy / numba are in the image):

    python oracle/build_ref.py            # or __graft_entry__.build()

oracle/_ref/ is git-ignored but travels to the GPU box with the repo snapshot,
so the GPU tests can run the reference's own driver (`run_with_state`) and
front end (`sylvadi.cli`) with the GPU bindings plugged in -- the drop-in
proof.  Only tests/ put oracle/_ref on sys.path; the product package imports
`sylvadi` only in its CLI adapter, from whatever installation the user has.
Nothing here copies reference sources into the repository.
"""

import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PKG = os.environ.get("SAD_REFERENCE_PKG", "/root/reference/pkg")
TARGET = os.path.join(HERE, "_ref")


def build(force=False, quiet=True):
    """Install the reference into oracle/_ref; returns the target or None when
    the reference tree is absent (the GPU box: it uses the shipped install)."""
    if not os.path.isdir(REF_PKG):
        return None
    stamp = os.path.join(TARGET, ".installed")
    if not force and os.path.exists(stamp):
        return TARGET
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(REF_PKG, src, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
        staging = os.path.join(tmp, "out")
        cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
               "--no-deps", "--target", staging, src]
        out = subprocess.run(cmd, capture_output=True, text=True)
        if out.returncode != 0:
            raise RuntimeError(f"pip install of the reference failed:\n{out.stderr[-2000:]}")
        if os.path.exists(TARGET):
            shutil.rmtree(TARGET)
        shutil.copytree(staging, TARGET)
    with open(stamp, "w") as fh:
        fh.write(REF_PKG + "\n")
    if not quiet:
        print(f"installed the reference into {TARGET}")
    return TARGET


if __name__ == "__main__":
    build(force="--force" in sys.argv, quiet=False)
