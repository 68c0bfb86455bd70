"""Build libpmg.so in-tree for sm_100a (B200) with nvcc.  Invoked by __graft_entry__.build()."""
import concurrent.futures
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpmg.so")
SOURCES = ["setup_host.cpp", "comm.cpp", "kernels.cu", "hot_kernels.cu", "star16.cu", "elem16.cu", "cr16.cu", "coarse_cg.cu", "ec_smoother.cu", "pmg_api.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-Xptxas", "-v"]


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def build(verbose=False, force=False, lib=None, extra=()):
    """lib / extra: experiment builds (another output name, extra -D flags); the product build
    is build() with the defaults."""
    LIB = lib or globals()["LIB"]
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    deps.append(os.path.join(HERE, "..", "include", "pmg.h"))
    if not force and os.path.exists(LIB) and all(os.path.getmtime(LIB) >= os.path.getmtime(d) for d in deps):
        return LIB
    objdir = os.path.join(HERE, "build" + ("_" + os.path.basename(LIB).replace(".so", "") if lib else ""))
    os.makedirs(objdir, exist_ok=True)
    def compile_one(s):
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        cmd = [_nvcc()] + ARCH + FLAGS + list(extra) + ["-x", "cu" if s.endswith(".cu") else "c++", "-c", s, "-o", o]
        return o, subprocess.run(cmd, capture_output=True, text=True)

    # translation units are independent: compile them concurrently
    with concurrent.futures.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        results = list(ex.map(compile_one, srcs))
    objs = []
    for s, (o, r) in zip(srcs, results):
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed on " + s)
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(o)
    cmd = [_nvcc()] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
