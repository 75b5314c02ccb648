"""Build libspconv.so in-tree with nvcc for sm_100a (B200). No JIT cache, no torch extension:
the library is a plain C-ABI shared object loaded with ctypes."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libspconv.so")
ROOT = os.path.dirname(HERE)

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2",
    "--expt-relaxed-constexpr",
    "-I", os.path.join(ROOT, "include"),
]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "spconv.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False, debug: bool = False,
          variant: str = "", defines=()) -> str:
    """debug=True builds libspconv_debug.so with -DSPC_DEBUG (device-side bounds reports);
    variant="name" with defines=("SPC_X", ...) builds libspconv_name.so (A/B experiments, loaded
    with SPC_LIB=...)."""
    if debug:
        variant, defines = "debug", tuple(defines) + ("SPC_DEBUG",)
    lib = LIB if not variant else os.path.join(HERE, f"libspconv_{variant}.so")
    if not force and not variant and not needs_build():
        return LIB
    objs = []
    bdir = os.path.join(HERE, "build" if not variant else f"build_{variant}")
    os.makedirs(bdir, exist_ok=True)
    procs = []
    for src in sources():
        obj = os.path.join(bdir, os.path.basename(src)[:-3] + ".o")
        cmd = [_nvcc(), "-c", src, "-o", obj] + NVCC_FLAGS + (["-Xptxas", "-v"] if ptxas_v else []) + \
              [f"-D{d}" for d in defines]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        if verbose or p.returncode != 0 or ptxas_v:
            sys.stdout.write(out.decode())
        if p.returncode != 0:
            failed.append(src)
    if failed:
        raise RuntimeError(f"nvcc failed for {failed}")
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([_nvcc(), "-shared", "-o", tmp] + objs +
                          ["-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC"])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv if a.startswith("-D")]
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), "")
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, ptxas_v="--ptxas" in sys.argv,
                debug="--debug" in sys.argv, variant=var, defines=defs))
