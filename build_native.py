"""Build every native artefact in-tree (sm_100a only).

    python build_native.py          # incremental
    python build_native.py --force

Targets
  paper_1703_00687_b200/libradsort.so   the product (CUDA kernels + C ABI, links NCCL)
  datagen/libradsort_datagen.so         seeded input generator (test/bench infra)
  verify/libradsort_verify.so           GPU result checkers (test/bench infra)
  oracle/liboracle.so                   CPU oracle (test infra; plain g++)
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_1703_00687_b200")
CSRC = os.path.join(PKG, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall"]
CUFLAGS += os.environ.get("RADSORT_NVCC_EXTRA", "").split()  # e.g. -DRADSORT_PHASE_PROF (profiling builds)


def _nccl_dirs():
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for p in spec.submodule_search_locations:
            cands.append(os.path.join(p, "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    raise RuntimeError("nccl.h from the nvidia-nccl wheel (the libnccl torch loads) not found")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd))
    return r


def build_radsort(force=False, verbose=False):
    target = os.path.join(PKG, "libradsort.so")
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + [
        os.path.join(ROOT, "include", "radsort.h")]
    units = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    if not force and not _stale(target, units + headers + [__file__]):
        return target
    inc, lib = _nccl_dirs()
    objdir = os.path.join(ROOT, "build")
    os.makedirs(objdir, exist_ok=True)

    def compile_one(u):
        o = os.path.join(objdir, os.path.basename(u) + ".o")
        if force or _stale(o, [u] + headers + [__file__]):
            cmd = [NVCC] + CUFLAGS + ["-I", inc, "-I", os.path.join(ROOT, "include"), "-c", u, "-o", o]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            _run(cmd)
        return o

    with ThreadPoolExecutor(max_workers=len(units)) as ex:
        objs = list(ex.map(compile_one, units))
    _run([NVCC] + ARCH + ["-shared", "-o", target] + objs +
         ["-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib])
    return target


def build_aux(force=False):
    out = []
    for src, target in ((os.path.join(ROOT, "datagen", "datagen.cu"), os.path.join(ROOT, "datagen", "libradsort_datagen.so")),
                        (os.path.join(ROOT, "verify", "verify.cu"), os.path.join(ROOT, "verify", "libradsort_verify.so"))):
        if force or _stale(target, [src, __file__]):
            _run([NVCC] + CUFLAGS + ["-shared", src, "-o", target])
        out.append(target)
    return out


def build_all(force=False, verbose=False):
    sys.path.insert(0, ROOT)
    from oracle import oracle as _oracle  # the checker is built, never used by the product

    with ThreadPoolExecutor(max_workers=3) as ex:
        f1 = ex.submit(build_radsort, force, verbose)
        f2 = ex.submit(build_aux, force)
        f3 = ex.submit(_oracle.build, force)
        return [f1.result()] + f2.result() + [f3.result()]


if __name__ == "__main__":
    for p in build_all(force="--force" in sys.argv, verbose="-v" in sys.argv):
        print(p)
