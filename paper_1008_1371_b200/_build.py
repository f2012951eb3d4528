"""In-tree build of libhsvd_b200.so for sm_100a (no JIT cache: the .so
travels with the repo snapshot to the GPU box)."""

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libhsvd_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
          "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr"]

def _nccl_include():
    """nccl.h of the NCCL torch loads (types only: the library is dlopen-ed)."""
    try:
        import nvidia.nccl
        for base in nvidia.nccl.__path__:
            inc = os.path.join(base, "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return inc
    except ImportError:
        pass
    return "/usr/include"


NCCL_INC = _nccl_include()

# translation unit -> extra flags.  The pointwise TU is the bit-exact mirror
# of the reference and must not contract a*b+c into FMA.
UNITS = {
    "hsvd_pointwise.cu": ["-fmad=false"],
    "hsvd_driver.cu": ["-fmad=false"],
    "hsvd_block.cu": [],
    "hsvd_sharded.cu": ["-I" + NCCL_INC],
    "hsvd_factor.cu": ["-fmad=false"],
}


def nvcc():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources_newer_than_lib():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    for f in os.listdir(CSRC):
        if os.path.getmtime(os.path.join(CSRC, f)) > t:
            return True
    hdr = os.path.join(HERE, "..", "include", "hsvd_b200.h")
    return os.path.getmtime(hdr) > t


def build(force=False, verbose=False):
    if not force and not sources_newer_than_lib():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    objs = []
    for src, extra in UNITS.items():
        obj = os.path.join(LIBDIR, src.replace(".cu", ".o"))
        cmd = [nvcc(), *ARCH, *COMMON, *extra, "-c", os.path.join(CSRC, src),
               "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        objs.append(obj)
    cmd = [nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-ldl"]
    subprocess.run(cmd, check=True)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
