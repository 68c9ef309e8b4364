"""Build libpnn.so (the CUDA path behind include/pnn.h) for sm_100a, in-tree.

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo, static cudart,
no fast-math (the fp32 path tracks the fp32 oracle).  NCCL is dlopen'ed at
run time (pnn_set_comm), so the library links no NCCL.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpnn.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale(out, deps):
    return not os.path.exists(out) or any(os.path.getmtime(d) > os.path.getmtime(out) for d in deps)


def build(force: bool = False, verbose: bool = False, extra=(), lib=None, objdir=None) -> str:
    """Compile csrc/*.cu into `lib` (default libpnn.so).  `extra` nvcc flags
    (e.g. -DPNN_SPIN_TAIL=1) build an experiment variant into its own lib/objdir."""
    LIB_OUT = lib or LIB
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) \
        + [os.path.join(ROOT, "include", "pnn.h")]
    if not force and not _stale(LIB_OUT, deps):
        return LIB_OUT
    objdir = objdir or os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    hdrs = [d for d in deps if not d.endswith(".cu")]
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + hdrs):
            cmd = [NVCC] + ARCH + FLAGS + list(extra) + ["-c", src, "-o", obj]
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stdout.write(out.decode())
        with open(os.path.join(objdir, os.path.basename(src) + ".ptxas.txt"), "wb") as f:
            f.write(out)
    tmp = LIB_OUT + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl"])
    os.replace(tmp, LIB_OUT)
    return LIB_OUT


if __name__ == "__main__":
    # python build.py [--force] [-v] [--variant NAME -DFLAG=1 ...]
    args = sys.argv[1:]
    if "--variant" in args:
        i = args.index("--variant")
        name = args[i + 1]
        flags = [a for a in args[i + 2:] if a.startswith("-D")]
        print(build(force=True, verbose="-v" in args, extra=flags,
                    lib=os.path.join(HERE, f"libpnn_{name}.so"), objdir=os.path.join(HERE, f"build_{name}")))
    else:
        print(build(force="--force" in args, verbose="-v" in args))
