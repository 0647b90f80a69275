"""Build libtpl.so in-tree: nvcc for sm_100a only, one shared cudart.

    python -m paper_1812_01108_b200.build        (or __graft_entry__.build())

The library links the CUDA runtime as a shared library (``-cudart shared``)
so that it uses the libcudart.so.12 PyTorch has already loaded in the
process; streams created by torch are therefore valid arguments.
"""
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtpl.so")
SOURCES = ["capi.cu", "backbone.cu", "fullatom.cu", "lrmsd.cu", "paper_baseline.cu", "segment.cu", "precise.cu", "packed.cu", "fused_lrmsd.cu"]
HEADERS = ["common.cuh", "kernels.h", "lrmsd_math.cuh", "packed.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-Xptxas", "-warn-spills", "-I" + os.path.join(ROOT, "include"),
    # accurate math: no --use_fast_math (precision)
    "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
]


def _nvcc():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a kernels")


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "tpl.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, profile_phases=False):
    """profile_phases=True builds build/libtpl_phases.so instead: the same
    kernels with %globaltimer stamps at phase boundaries (latency studies)."""
    lib_out = LIB
    flags = list(NVCC_FLAGS)
    if profile_phases:
        lib_out = os.path.join(HERE, "build", "libtpl_phases.so")
        flags.append("-DTPL_PROFILE_PHASES")
        force = True
    if not force and not _stale():
        return LIB
    nvcc = _nvcc()
    objdir = os.path.join(HERE, "build", "phases" if profile_phases else "obj")
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [nvcc] + flags + ["-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = lib_out + ".tmp"
    cmd = [nvcc] + ARCH + ["-shared", "-cudart", "shared", "-o", tmp] + objs
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib_out)
    return lib_out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, profile_phases="--phases" in sys.argv))
