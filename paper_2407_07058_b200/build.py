"""Build libappd.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2407_07058_b200.build

No --use_fast_math: the points-mode distance chain (R1) must be IEEE round to
nearest with no denormal flushing; the kernels also use explicit
__fsub_rn / __fmaf_rn so contraction cannot change it.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libappd.so")
# development build (-DAPPD_DEV_HOOKS: debug prints, experiments, APPD_SYNC_EACH); never the
# product library -- tools load it explicitly through APPD_LIB
DEV_LIB = os.path.join(LIBDIR, "libappd_dev.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nccl_include() -> str:
    try:
        import nvidia.nccl  # noqa: F401

        base = os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
    except Exception:  # pragma: no cover
        base = "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl"
    return os.path.join(base, "include")


FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xptxas", "-warn-spills",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "appd.h"), __file__]
    return all(os.path.getmtime(p) <= t for p in deps)


def build(force: bool = False, verbose: bool = False, dev: bool = False) -> str:
    """Compile every source to an object in parallel (nvcc -dc is not needed: no device
    linking across files), then link libappd.so (dev: libappd_dev.so)."""
    lib = DEV_LIB if dev else LIB
    if not force and up_to_date(lib):
        return lib
    from concurrent.futures import ThreadPoolExecutor

    os.makedirs(LIBDIR, exist_ok=True)
    objdir = os.path.join(LIBDIR, "obj_dev" if dev else "obj")
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", nccl_include()]
    cflags = [f for f in FLAGS if f != "-shared"] + (["-DAPPD_DEV_HOOKS"] if dev else [])

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *cflags, *inc, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, end="", flush=True)
        return obj

    srcs = sources()
    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, srcs))
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC", *objs,
           "-o", lib + ".tmp", "-ldl"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, dev="--dev" in sys.argv))
