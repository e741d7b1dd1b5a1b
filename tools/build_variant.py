"""Build an A/B variant of the library with extra -D defines into
tools/bin_<name>.so (git-ignored; ships to the GPU box), for SAD_LIB_PATH runs.

    python tools/build_variant.py NAME -DSAD_KB1=9 [-D...]
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_02891_b200 import _build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
objdir = os.path.join(b.REPO, "build", "variant_" + name)
os.makedirs(objdir, exist_ok=True)
nv = b.nvcc()


def comp(u):
    uname, src, d = u
    obj = os.path.join(objdir, uname + ".o")
    cmd = [nv] + b.NVCC_FLAGS + d + defs + ["-c", "-o", obj, os.path.join(b.SRC_DIR, src)]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode:
        raise RuntimeError(p.stderr[-3000:])
    return obj


with ThreadPoolExecutor(max_workers=os.cpu_count()) as ex:
    objs = list(ex.map(comp, b.UNITS))
out = os.path.join(b.REPO, "tools", f"bin_{name}.so")
subprocess.run([nv] + b.ARCH + ["-shared", "-o", out] + objs + ["-ldl"], check=True)
print("built", out)
