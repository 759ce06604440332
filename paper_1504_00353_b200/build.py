"""Build libpolar.so in-tree: emit the unrolled decoders, compile them for sm_100a, link.

Steps (all native; nothing here computes the method):
  1. g++: csrc/codegen.cpp + csrc/construct.cpp -> build/polar_codegen
  2. polar_codegen codes.txt + codes_random.txt -> build/gen/code_<name>.cu, registry.cpp
  3. nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo: every .cu -> .o (parallel,
     skipped when the source and headers are unchanged)
  4. nvcc -shared -> paper_1504_00353_b200/libpolar.so
"""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
# Experiment builds (tools/variant_build.sh) redirect these; the product build uses the defaults.
BUILD = os.environ.get("POLAR_BUILD_DIR", os.path.join(PKG, "build"))
GEN = os.path.join(BUILD, "gen")
OBJ = os.path.join(BUILD, "obj")
LIB = os.environ.get("POLAR_LIB_OUT", os.path.join(PKG, "libpolar.so"))
SPEC_FILES = os.environ.get("POLAR_CODES", "codes.txt,codes_random.txt").split(",")
EXTRA = os.environ.get("POLAR_NVCC_EXTRA", "").split()
INCLUDE = os.path.join(os.path.dirname(PKG), "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-I", CSRC, "-I", INCLUDE,
                  "-Xptxas", "-v", "--resource-usage"] + EXTRA
HEADERS = ["decoder.cuh", "kernels.cuh", "xframe.cuh", "registry.hpp", "tree.hpp"]


def _run(cmd, log=None):
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if log:
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + r.stdout)
    if r.returncode != 0:
        raise RuntimeError(f"command failed ({r.returncode}): {' '.join(cmd)}\n{r.stdout[-4000:]}")
    return r.stdout


def _digest(paths, extra=""):
    h = hashlib.sha256(extra.encode())
    for p in paths:
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def _compile(src, obj, flags):
    deps = [src] + [os.path.join(CSRC, x) for x in HEADERS]
    stamp = obj + ".sha"
    d = _digest(deps, " ".join(flags))
    if os.path.exists(obj) and os.path.exists(stamp) and open(stamp).read() == d:
        return False
    _run([NVCC, *flags, "-c", src, "-o", obj], log=obj + ".log")
    with open(stamp, "w") as f:
        f.write(d)
    return True


def build_one(build_dir: str, lib_out: str, spec_files, extra, verbose: bool = True, jobs: int | None = None) -> str:
    GEN, OBJ, LIB = os.path.join(build_dir, "gen"), os.path.join(build_dir, "obj"), lib_out
    nvflags = NVFLAGS + list(extra)
    os.makedirs(GEN, exist_ok=True)
    os.makedirs(OBJ, exist_ok=True)
    # 1. the emitter
    gen_exe = os.path.join(build_dir, "polar_codegen")
    gsrc = [os.path.join(CSRC, "codegen.cpp"), os.path.join(CSRC, "construct.cpp"), os.path.join(CSRC, "tree.hpp")]
    gstamp = gen_exe + ".sha"
    gd = _digest(gsrc)
    if not (os.path.exists(gen_exe) and os.path.exists(gstamp) and open(gstamp).read() == gd):
        _run(["g++", "-O2", "-std=c++17", "-I", CSRC, gsrc[0], gsrc[1], "-o", gen_exe])
        with open(gstamp, "w") as f:
            f.write(gd)
    # 2. emit into a scratch dir, then replace only the files whose content changed
    spec = os.path.join(build_dir, "codes_all.txt")
    with open(spec, "w") as f:
        for name in spec_files:
            p = name if os.path.isabs(name) else os.path.join(PKG, name)
            if os.path.exists(p):
                f.write(open(p).read() + "\n")
    scratch = GEN + ".new"
    shutil.rmtree(scratch, ignore_errors=True)
    os.makedirs(scratch)
    _run([gen_exe, spec, scratch])
    new = set(os.listdir(scratch))
    for fn in os.listdir(GEN):
        if fn not in new:
            os.remove(os.path.join(GEN, fn))
    for fn in new:
        src, dst = os.path.join(scratch, fn), os.path.join(GEN, fn)
        if not (os.path.exists(dst) and open(dst).read() == open(src).read()):
            shutil.copyfile(src, dst)
    shutil.rmtree(scratch)
    # 3. compile
    units = [(os.path.join(CSRC, "polar_api.cu"), "polar_api.o"),
             (os.path.join(CSRC, "generic.cu"), "generic.o"),
             (os.path.join(CSRC, "construct.cpp"), "construct.o"),
             (os.path.join(GEN, "registry.cpp"), "registry.o")]
    units += [(os.path.join(GEN, fn), fn[:-3] + ".o") for fn in sorted(new) if fn.endswith(".cu")]
    jobs = jobs or max(1, os.cpu_count() or 1)

    def one(u):
        src, o = u
        flags = nvflags if src.endswith(".cu") else [f for f in nvflags if f not in ("-Xptxas", "-v", "--resource-usage")]
        t = _compile(src, os.path.join(OBJ, o), flags)
        if t and verbose:
            print(f"[polar build] compiled {os.path.basename(src)}", flush=True)
        return t

    with ThreadPoolExecutor(jobs) as ex:
        changed = any(list(ex.map(one, units)))
    objs = [os.path.join(OBJ, o) for _, o in units]
    if changed or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        tmp = LIB + f".tmp{os.getpid()}"
        _run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"])
        os.replace(tmp, LIB)
        if verbose:
            print(f"[polar build] linked {LIB}", flush=True)
    return LIB


def build(verbose: bool = True, jobs: int | None = None) -> str:
    """The product library (every code of codes.txt + codes_random.txt)."""
    return build_one(BUILD, LIB, SPEC_FILES, [], verbose, jobs)


def build_dump(verbose: bool = True, jobs: int | None = None) -> str:
    """libpolar_dump.so: the same kernels built with POLAR_DEBUG_DUMP for the codes of
    codes_dump.txt -- test infrastructure recording every F/G output (alpha stage) so that the
    GPU's intermediate LLRs can be compared with the oracle's (tests/test_alpha_dump.py)."""
    return build_one(os.path.join(PKG, "build_dump"), os.path.join(PKG, "libpolar_dump.so"), ["codes_dump.txt"],
                     ["-DPOLAR_DEBUG_DUMP"], verbose, jobs)


if __name__ == "__main__":
    build(jobs=int(sys.argv[1]) if len(sys.argv) > 1 else None)
    if os.environ.get("POLAR_BUILD_DUMP", "1") != "0":
        build_dump(jobs=int(sys.argv[1]) if len(sys.argv) > 1 else None)
