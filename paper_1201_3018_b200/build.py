"""Build libpackedconv.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels
with the repo snapshot to the GPU box)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("pc_kernels.cu", "pc_tiled.cu", "pc_fft.cu", "pc_api.cu")]
DEPS = SOURCES + [os.path.join(HERE, "csrc", f) for f in ("pc_device.cuh", "pc_kernels.h", "pc_intfp.cuh")] + \
    [os.path.join(ROOT, "include", "packedconv.h")]
OUT = os.path.join(HERE, "libpackedconv.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
EXTRA = os.environ.get("PC_NVCC_EXTRA", "").split()
FLAGS = EXTRA + ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v"]
OBJ_DIR = os.path.join(HERE, "build")


def up_to_date():
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def _compile(src):
    obj = os.path.join(OBJ_DIR, os.path.basename(src)[:-3] + ".o")
    res = subprocess.run([NVCC] + FLAGS + ["-c", "-o", obj, src], capture_output=True, text=True)
    return obj, res


def build_library(force=False, verbose=False):
    """nvcc -c of every source in parallel (one process each), then one shared-library link
    with the static CUDA runtime."""
    if not force and up_to_date():
        return OUT
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(OBJ_DIR, exist_ok=True)
    with ThreadPoolExecutor(len(SOURCES)) as ex:
        results = list(ex.map(_compile, SOURCES))
    for obj, res in results:
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc failed: " + obj)
        if verbose:
            sys.stderr.write(res.stderr)
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-o", OUT] + \
        [obj for obj, _ in results]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed")
    return OUT


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose=True))
