"""Build libsylvadi_b200.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2312_02891_b200._build [--force] [-j N]

The library is several translation units compiled in parallel (the host
runtime + C-ABI, and one unit per variant of the persistent GMRES kernel),
then linked with nvcc into one shared object.  Objects go to build/ (ignored
by git); the .so is written next to this file so it travels with the repo
snapshot to the GPU box.
"""

import glob
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

_HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(_HERE)
SRC_DIR = os.path.join(_HERE, "csrc")
OBJ_DIR = os.path.join(REPO, "build", "sylvadi_b200")
N_COOP_VARIANTS = 10   # SAD_COOP_VARIANTS in sad_coop.cuh

# (object name, source, extra defines)
UNITS = [("sad_capi", "sad_capi.cu", [])] + [
    (f"sad_spmm_{p}", "sad_spmm_launch.cu", [f"-DSAD_SPMM_PART={p}"]) for p in range(4)] + [
    (f"sad_coop_{v}", "sad_coop.cu", [f"-DSAD_COOP_VARIANT={v}"]) for v in range(N_COOP_VARIANTS)] + [
    (f"sad_bicg_{p}", "sad_bicg.cu", [f"-DSAD_BICG_PART={p}"]) for p in range(2)] + [
    (f"sad_minres_{p}", "sad_minres.cu", [f"-DSAD_MINRES_PART={p}"]) for p in range(2)] + [
    ("sad_precond", "sad_precond.cu", [])]
HEADERS = sorted(glob.glob(os.path.join(SRC_DIR, "*.cuh"))) + [
    os.path.join(REPO, "include", "sylvadi_b200.h")]
DEPS = [os.path.join(SRC_DIR, s) for s in {u[1] for u in UNITS}] + HEADERS
OUT = os.path.join(_HERE, "libsylvadi_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def nvcc():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths)


def up_to_date():
    if not os.path.exists(OUT):
        return False
    return _newest(DEPS) <= os.path.getmtime(OUT)


def _compile(unit, nv):
    name, src, defs = unit
    obj = os.path.join(OBJ_DIR, name + ".o")
    deps = [os.path.join(SRC_DIR, src)] + HEADERS
    if os.path.exists(obj) and _newest(deps) <= os.path.getmtime(obj):
        return obj, 0, ""
    cmd = [nv] + NVCC_FLAGS + defs + ["-c", "-o", obj, os.path.join(SRC_DIR, src)]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    return obj, proc.returncode, " ".join(cmd) + "\n" + proc.stdout + proc.stderr


def build(force=False, verbose=False, jobs=None):
    if not force and up_to_date():
        return OUT
    os.makedirs(OBJ_DIR, exist_ok=True)
    if force:
        for o in glob.glob(os.path.join(OBJ_DIR, "*.o")):
            os.remove(o)
    nv = nvcc()
    jobs = jobs or max(1, min(len(UNITS), os.cpu_count() or 1))
    with ThreadPoolExecutor(max_workers=jobs) as ex:
        results = list(ex.map(lambda u: _compile(u, nv), UNITS))
    log_path = os.path.join(SRC_DIR, "build.log")
    with open(log_path, "w") as fh:
        for _, _, log in results:
            fh.write(log)
    bad = [(o, rc, log) for o, rc, log in results if rc != 0]
    if bad:
        raise RuntimeError(f"nvcc failed for {[os.path.basename(o) for o, _, _ in bad]}; "
                           f"see {log_path}\n" + bad[0][2][-4000:])
    cmd = [nv] + ARCH + ["-shared", "-o", OUT] + [o for o, _, _ in results] + ["-ldl"]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError("link failed:\n" + proc.stderr[-4000:])
    if verbose:
        print(f"built {OUT}")
    return OUT


if __name__ == "__main__":
    j = None
    if "-j" in sys.argv:
        j = int(sys.argv[sys.argv.index("-j") + 1])
    build(force="--force" in sys.argv, verbose=True, jobs=j)
