"""In-tree build of libamgcu.so (sm_100a) and of the CPU oracles.

nvcc flags: -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 --fmad=false.
--fmad=false (and -ffp-contract=off for host code) keeps every multiply and
add separately rounded, which the bit-exact parity with the reference's CPU
code requires (SURVEY.md §7 "Compile flags").
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
OBJDIR = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(LIBDIR, "libamgcu.so")

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-lineinfo", "-O3", "--fmad=false", "-std=c++20", "--expt-relaxed-constexpr",
                     "-Xcompiler", "-fPIC,-ffp-contract=off,-O3", "-I" + os.path.join(ROOT, "include")]
CXX_FLAGS = ["-O3", "-std=gnu++20", "-fPIC", "-ffp-contract=off", "-I" + os.path.join(ROOT, "include")]

CU_SOURCES = ["primitives.cu", "sparse_core.cu", "blas.cu", "seqsum.cu", "strength.cu", "aggregate.cu", "relax.cu", "relax_more.cu", "arnoldi.cu",
              "interp.cu", "setup.cu", "cycle.cu", "capi.cu"]
CXX_SOURCES = ["problems.cpp"]
# every header in csrc (a header edit must rebuild its includers)
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h")))


def _digest(paths):
    h = hashlib.sha256()
    for p in paths:
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stderr


def build_lib(force=False, jobs=8, verbose=False):
    os.makedirs(LIBDIR, exist_ok=True)
    os.makedirs(OBJDIR, exist_ok=True)
    hdr = _digest([os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "amgcu.h")])
    tasks = []
    objs = []
    for src in CU_SOURCES + CXX_SOURCES:
        path = os.path.join(CSRC, src)
        key = _digest([path]) + hdr
        obj = os.path.join(OBJDIR, f"{src}.{key}.o")
        objs.append(obj)
        if os.path.exists(obj) and not force:
            continue
        if src.endswith(".cu"):
            cmd = [NVCC] + NVCC_FLAGS + ["-c", path, "-o", obj]
        else:
            cmd = ["g++"] + CXX_FLAGS + ["-c", path, "-o", obj]
        tasks.append(cmd)
    if tasks:
        with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
            for err in ex.map(_run, tasks):
                if verbose and err:
                    sys.stderr.write(err)
    tmp = LIB + ".tmp"
    if tasks or not os.path.exists(LIB) or force:
        _run([NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart_static", "-L" + os.path.join(CUDA_HOME, "lib64"), "-lcusolver"])
        os.replace(tmp, LIB)
    # keep only this build's objects (the cache is content-hashed, stale ones pile up)
    keep = set(objs)
    for f in os.listdir(OBJDIR):
        full = os.path.join(OBJDIR, f)
        if f.endswith(".o") and full not in keep:
            os.remove(full)
    return LIB


def build_oracle(force=False):
    """CPU oracles (test infrastructure): the restatement, and -- when the
    reference tree is present -- the reference headers against the Eigen
    stand-in (oracle/_ref)."""
    odir = os.path.join(ROOT, "oracle")
    out = os.path.join(odir, "build", "liboracle_port.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    srcs = [os.path.join(odir, "rnamg_port.cpp"), os.path.join(odir, "oracle_abi.h"),
            os.path.join(CSRC, "small_dense.h"), os.path.join(ROOT, "include", "amgcu.h")]
    stamp = out + ".stamp"
    key = _digest(srcs)
    if force or not os.path.exists(out) or not os.path.exists(stamp) or open(stamp).read() != key:
        _run(["g++", "-O3", "-std=gnu++20", "-ffp-contract=off", "-fPIC", "-shared",
              os.path.join(odir, "rnamg_port.cpp"), "-o", out + ".tmp"])
        os.replace(out + ".tmp", out)
        with open(stamp, "w") as f:
            f.write(key)
    # the config generators as a CPU library of their own (the reference arm's inputs)
    gen = os.path.join(odir, "build", "libconfiggen.so")
    gsrcs = [os.path.join(odir, "config_gen.cpp"), os.path.join(CSRC, "problems.cpp"),
             os.path.join(CSRC, "host_common.h"), os.path.join(ROOT, "include", "amgcu.h")]
    gstamp = gen + ".stamp"
    gkey = _digest(gsrcs)
    if force or not os.path.exists(gen) or not os.path.exists(gstamp) or open(gstamp).read() != gkey:
        _run(["g++"] + CXX_FLAGS + ["-shared", gsrcs[0], gsrcs[1], "-o", gen + ".tmp"])
        os.replace(gen + ".tmp", gen)
        with open(gstamp, "w") as f:
            f.write(gkey)
    ref_root = os.environ.get("AMG_REFERENCE_ROOT", "/root/reference")
    ref_so = os.path.join(odir, "_ref", "libamgref.so")
    if os.path.isdir(os.path.join(ref_root, "proj", "include", "amg")):
        rstamp = ref_so + ".stamp"
        rkey = _digest([os.path.join(odir, "ref_entry.cpp"), os.path.join(odir, "eigen_shim", "Eigen", "Dense"),
                        os.path.join(CSRC, "small_dense.h")])
        if force or not os.path.exists(ref_so) or not os.path.exists(rstamp) or open(rstamp).read() != rkey:
            _run(["bash", os.path.join(odir, "build_ref.sh")])
            with open(rstamp, "w") as f:
                f.write(rkey)
    return out


if __name__ == "__main__":
    force = "--force" in sys.argv
    print(build_lib(force=force, verbose=True))
    print(build_oracle(force=force))
