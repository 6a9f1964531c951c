"""Build librid.so (the C-ABI library of include/rid.h) in-tree for sm_100a with nvcc.

    python -m paper_1205_3830_b200.build [--force] [--experiments]

The .so lands next to this file so it travels with the repo snapshot to the GPU box.
--experiments (or RID_BUILD_EXPERIMENTS=1) compiles with -DRID_EXPERIMENTS, which makes the
tuning knobs of the tools/ scripts (tile shapes, ring depths, ...; rid_host.h experiment_env)
effective; the product build ignores them.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librid.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import nvidia.nccl  # the NCCL 2.28 that torch also loads

    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  [os.path.join(ROOT, "include", "rid.h")])


STAMP = os.path.join(ROOT, "build", "rid_obj", "flags.txt")


def _flags(experiments: bool):
    return ["-DRID_EXPERIMENTS"] if experiments else []


def up_to_date(experiments: bool = False) -> bool:
    if not os.path.exists(LIB):
        return False
    try:
        with open(STAMP) as f:
            if f.read() != " ".join(_flags(experiments)):
                return False
    except OSError:
        # no stamp (a fresh snapshot): the shipped .so is a product build
        if experiments:
            return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in sources() + headers() + [__file__])


def build(force: bool = False, verbose: bool = False, experiments: bool | None = None) -> str:
    if experiments is None:
        experiments = os.environ.get("RID_BUILD_EXPERIMENTS", "0") not in ("", "0")
    if not force and up_to_date(experiments):
        return LIB
    inc, libdir = _nccl_dirs()
    objdir = os.path.join(ROOT, "build", "rid_obj")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-Xptxas", "-v" if verbose else "-O3", "--expt-relaxed-constexpr", *_flags(experiments),
               "-I", inc, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                            text=True)))
        objs.append(obj)
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(out)
        failed |= p.returncode != 0
    if failed:
        raise RuntimeError("nvcc failed")
    tmp = LIB + ".tmp"
    link = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-L", libdir, "-l:libnccl.so.2",
            f"-Xlinker=-rpath={libdir}", "-lcudart"]
    subprocess.check_call(link)
    os.replace(tmp, LIB)
    with open(STAMP, "w") as f:
        f.write(" ".join(_flags(experiments)))
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv,
          experiments=True if "--experiments" in sys.argv else None)
    print(LIB)
