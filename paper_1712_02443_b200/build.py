"""Build the in-tree CUDA library libaim_b200.so for sm_100a (nvcc, no JIT)."""
from __future__ import annotations

import hashlib
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libaim_b200.so")
SOURCES = ["aim_api.cu", "k_plan.cu", "k_fft.cu", "k_matvec.cu", "k_gmres.cu", "k_slab.cu", "k_precond.cu",
           "k_reduced.cu", "k_compress.cu", "k_near_stream.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "--expt-relaxed-constexpr"]


def _key(deps, defines, flags):
    """Cache key of a build: the sources' contents, the defines and the flags."""
    h = hashlib.sha256()
    for d in sorted(deps):
        h.update(d.encode())
        with open(d, "rb") as f:
            h.update(f.read())
    h.update(json.dumps([list(defines), list(flags)]).encode())
    return h.hexdigest()


def build(verbose: bool = False, force: bool = False, out: str | None = None, defines=()) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    deps.append(os.path.join(HERE, "..", "include", "aim.h"))
    lib = out or LIB
    stamp = lib + ".buildkey"
    key = _key(deps, defines, FLAGS)
    if not force and os.path.exists(lib) and os.path.exists(stamp) and open(stamp).read() == key:
        return lib
    objs = [os.path.join(CSRC, os.path.basename(s).replace(".cu", f".{os.getpid()}.o")) for s in srcs]
    try:
        procs = []
        for s, o in zip(srcs, objs):
            cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-c", s, "-o", o]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True), s))
        err = False
        for pr, s in procs:
            log, _ = pr.communicate()
            if pr.returncode != 0:
                err = True
                sys.stderr.write(f"nvcc failed for {s}:\n{log}\n")
            elif verbose and log:
                sys.stderr.write(log)
        if err:
            raise RuntimeError("CUDA build failed")
        subprocess.run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", lib, *objs, "-lcudart"],
                       check=True)
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    with open(stamp, "w") as f:
        f.write(key)
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True))
