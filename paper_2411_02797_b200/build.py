"""Builds libdc.so (the C-ABI CUDA library) in-tree for sm_100a."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libdc.so")
SOURCES = ["capi.cu", "intern.cu", "build.cu", "columns.cu", "pc.cu", "pc_owner.cu", "views.cu", "merge.cu", "rules.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    try:
        import nvidia.nccl
        base = list(nvidia.nccl.__path__)[0]
        return os.path.join(base, "include"), os.path.join(base, "lib")
    except Exception:
        return None, None


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))]
    deps.append(os.path.join(ROOT, "include", "dc.h"))
    if not force and os.path.exists(SO) and os.path.getmtime(SO) >= max(os.path.getmtime(p) for p in deps):
        return SO
    objdir = os.path.join(HERE, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    inc, lib = nccl_paths()
    flags = ["-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include")]
    if inc:
        flags += ["-I", inc, "-DDC_HAVE_NCCL=1"]
    flags += ["-Xptxas", "-v"] if verbose else []
    from concurrent.futures import ThreadPoolExecutor

    def one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(p) for p in deps if not p.endswith(".cu") or p == src):
            subprocess.check_call(["nvcc", *flags, "-c", src, "-o", obj])
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(one, srcs))
    link = ["nvcc", "-shared", *ARCH, "-o", SO + ".tmp", *objs]
    if lib:
        link += ["-L", lib, "-l:libnccl.so.2", f"-Xlinker", f"-rpath={lib}"]
    subprocess.check_call(link)
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO)
