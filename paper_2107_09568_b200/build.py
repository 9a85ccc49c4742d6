"""Build libiga.so in-tree with nvcc for sm_100a (no JIT, no torch extension)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libiga.so")
SOURCES = ["host_build.cpp", "iga_api.cu", "kernels_tables.cu", "kernels_macro.cu", "kernels_gemm.cu",
           "kernels_scatter.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-fopenmp,-O3", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def build(verbose=False, force=False, defines=(), lib=None):
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    deps.append(os.path.join(HERE, "..", "include", "iga.h"))
    LIBP = lib or LIB
    if not force and os.path.exists(LIBP) and all(os.path.getmtime(LIBP) >= os.path.getmtime(d) for d in deps):
        return LIBP
    objdir = os.path.join(HERE, "build" if not defines else "build_" + "_".join(defines))
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, os.path.basename(src) + ".o") for src in srcs]

    def compile_one(src_obj):
        src, obj = src_obj
        cmd = [NVCC] + FLAGS + ["-D" + x for x in defines] + ["-c", src, "-o", obj]
        return src, subprocess.run(cmd, capture_output=True, text=True)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(srcs)) as ex:   # nvcc processes in parallel
        for src, r in ex.map(compile_one, zip(srcs, objs)):
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed for {src}")
            if verbose:
                sys.stderr.write(r.stderr)
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIBP] + objs + ["-lgomp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    return LIBP


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
