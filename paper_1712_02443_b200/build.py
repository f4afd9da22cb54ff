"""Build the in-tree CUDA library libaim_b200.so for sm_100a (nvcc, no JIT)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libaim_b200.so")
SOURCES = ["aim_api.cu", "k_plan.cu", "k_fft.cu", "k_matvec.cu", "k_gmres.cu", "k_slab.cu", "k_precond.cu", "k_reduced.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "--expt-relaxed-constexpr"]


def build(verbose: bool = False, force: bool = False, out: str | None = None, defines=()) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    deps.append(os.path.join(HERE, "..", "include", "aim.h"))
    lib = out or LIB
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= max(os.path.getmtime(d) for d in deps):
        return lib
    objs = []
    procs = []
    for s in srcs:
        o = os.path.join(CSRC, os.path.basename(s).replace(".cu", f".{os.getpid()}.o"))
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-c", s, "-o", o]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True), s))
        objs.append(o)
    err = False
    for pr, s in procs:
        out, _ = pr.communicate()
        if pr.returncode != 0:
            err = True
            sys.stderr.write(f"nvcc failed for {s}:\n{out}\n")
        elif verbose and out:
            sys.stderr.write(out)
    if err:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
        raise RuntimeError("CUDA build failed")
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", lib, *objs, "-lcudart"]
    subprocess.run(cmd, check=True)
    for o in objs:
        os.remove(o)
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True))
