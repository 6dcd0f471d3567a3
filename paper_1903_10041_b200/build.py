"""Build libadmm_b200.so in-tree with nvcc for sm_100a (no JIT, no torch
extension machinery): the .so travels to the GPU box with the repo snapshot."""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libadmm_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import nvidia.nccl

    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(ROOT, "include", "admm.h")])


def up_to_date() -> bool:
    if not os.path.exists(SO):
        return False
    t = os.path.getmtime(SO)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile every csrc/*.cu translation unit (in parallel) and link the shared
    library.  out/defines: experimental variants (e.g. -DSWEEP2_MINB=3) written next
    to the product library and loaded with ADMM_SO=<path>; the product build takes
    neither."""
    SO = out or globals()["SO"]
    if not out and not force and up_to_date():
        return SO
    inc, lib = nccl_dirs()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    odir = os.path.join(HERE, "build", "obj" if not out else "obj_" + os.path.basename(out))
    os.makedirs(odir, exist_ok=True)
    common = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc,
              *[f"-D{d}" for d in defines]]
    if verbose:
        common.insert(1, "-Xptxas=-v")
    units = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "admm.h"), __file__]
    hdr_t = max(os.path.getmtime(h) for h in headers)
    procs, objs = [], []
    for u in units:
        o = os.path.join(odir, os.path.basename(u)[:-3] + ".o")
        objs.append(o)
        # an object is reused when it is newer than its unit and every header (any unit
        # may include any header) and was built with the same flags
        flags_file = o + ".flags"
        same_flags = os.path.exists(flags_file) and open(flags_file).read() == " ".join(common)
        if (not force and same_flags and os.path.exists(o)
                and os.path.getmtime(o) >= max(hdr_t, os.path.getmtime(u))):
            continue
        open(flags_file, "w").write(" ".join(common))
        procs.append((u, subprocess.Popen(common + ["-c", "-o", o, u], stdout=subprocess.PIPE,
                                          stderr=subprocess.PIPE, text=True)))
    failed = False
    for u, p in procs:
        so, se = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(f"--- {u}\n" + so + se)
            failed = True
        elif verbose:
            sys.stderr.write(se)
    if failed:
        raise RuntimeError("nvcc failed building libadmm_b200.so")
    link = [nvcc, *ARCH, "-shared", "-o", SO + ".tmp", *objs,
            "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{lib}"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libadmm_b200.so")
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("-D", action="append", default=[])
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.v, out=a.out, defines=a.D))
