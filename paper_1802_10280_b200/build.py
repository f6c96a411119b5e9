"""Build libescoin.so (the method's C-ABI library).

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo; IEEE fp32 (no
--use_fast_math, no FTZ: reading R#22).  cudart is linked statically so the
library does not depend on which libcudart the host process (torch) loaded.
Objects are rebuilt only when a source or header is newer; variants compile
in parallel (each register-tiled variant is a large generated kernel).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
GEN = os.path.join(CSRC, "generated")
OBJ = os.path.join(ROOT, "build", "obj")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libescoin.so")
# in-process PTX compiler for the pattern-specialised kernels (jit_sconv.cpp)
_LIB64 = os.path.join(os.path.dirname(os.path.dirname(os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc"))), "lib64")
PTXC = os.path.join(_LIB64, "libnvptxcompiler_static.a")
# (the device linker for multi-unit specialised kernels, nvJitLink, is dlopen'ed at run time)

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-I", INCLUDE, "-I", CSRC,
                 "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, headers):
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    log = obj + ".log"
    if _newer(obj, [src] + headers):
        tmp = obj + ".tmp"
        with open(log, "w") as lf:
            subprocess.check_call([NVCC] + CFLAGS + ["-c", src, "-o", tmp], stdout=lf, stderr=subprocess.STDOUT)
        os.replace(tmp, obj)
    return obj


def _link(out, objs, libs):
    if _newer(out, objs):
        tmp = out + ".tmp"
        subprocess.check_call([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs + libs)
        os.replace(tmp, out)


def build(jobs: int | None = None, verbose: bool = False) -> str:
    sys.path.insert(0, CSRC)
    try:
        import gen_sconv
    finally:
        sys.path.pop(0)
    variants = gen_sconv.main(GEN)
    os.makedirs(OBJ, exist_ok=True)
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(INCLUDE, "*.h")) + [os.path.join(GEN, "variants_table.inc")]
    core = [os.path.join(CSRC, "escoin_host.cu"), os.path.join(CSRC, "sconv_paper.cu"),
            os.path.join(CSRC, "stretch_device.cu"), os.path.join(CSRC, "dense_tc.cu"),
            os.path.join(CSRC, "jit_sconv.cpp")]
    srcs = core + variants
    jobs = jobs or max(1, min(len(srcs), os.cpu_count() or 4))
    with ThreadPoolExecutor(jobs) as ex:
        objs = dict(zip(srcs, ex.map(lambda s: _compile(s, headers), srcs)))
    _link(LIB, [objs[s] for s in core + variants], [PTXC, "-ldl"])
    if verbose:
        for s in srcs:
            log = os.path.join(OBJ, os.path.basename(s) + ".o.log")
            if os.path.exists(log):
                print(open(log).read())
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
