"""In-tree build of the CUDA library (sm_100a) -> paper_2003_04776_b200/libzz.so.

Each translation unit is compiled in parallel (nvcc -c), then linked with nvcc -shared.
The ptxas register/spill report is kept in csrc/ptxas.log."""
import concurrent.futures
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libzz.so")
SRCS = ["zz_api.cu", "zz_kernels.cu", "zz_update.cu", "zz_diag3.cu", "zz_back.cu", "zz_left.cu", "zz_complex.cu", "zz_comm.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v"]
OBJDIR = os.path.join(HERE, "build")


def _stale():
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))
            if f.endswith((".cu", ".cuh", ".h"))]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "zz.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src):
    obj = os.path.join(OBJDIR, os.path.basename(src) + ".o")
    r = subprocess.run([NVCC] + FLAGS + ["-c", "-o", obj, src], capture_output=True, text=True)
    return src, obj, r


def build(force=False, verbose=False):
    if not force and not _stale():
        return SO
    os.makedirs(OBJDIR, exist_ok=True)
    srcs = [os.path.join(HERE, "csrc", f) for f in SRCS]
    with concurrent.futures.ThreadPoolExecutor(len(srcs)) as ex:
        results = list(ex.map(_compile, srcs))
    log = []
    for src, obj, r in results:
        if r.returncode != 0:
            raise RuntimeError("nvcc failed on %s:\n%s%s" % (src, r.stdout, r.stderr))
        log.append(r.stderr)
    objs = [obj for _, obj, _ in results]
    cudalib = os.path.join(os.path.dirname(os.path.dirname(NVCC)), "lib64")
    r = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", SO + ".tmp"] + objs
                       + ["-L" + cudalib, "-ldl", "-Xlinker", "-rpath", "-Xlinker", cudalib],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + r.stdout + r.stderr)
    if verbose:
        print("".join(log))
    with open(os.path.join(HERE, "csrc", "ptxas.log"), "w") as f:
        f.write("".join(log))
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    build(force=True, verbose=True)
