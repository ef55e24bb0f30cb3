"""Build libsnx.so (the sm_100a kernels + C ABI) in-tree with nvcc.

The shared object lands in paper_1802_09113_b200/_lib/ so it travels with the
repo snapshot to the GPU box; nothing is JIT-compiled at run time.
"""

import glob
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIBPATH = os.path.join(LIBDIR, "libsnx.so")
INCLUDE = os.path.join(ROOT, "include")
OBJDIR = os.path.join(ROOT, "build", "obj")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# cuBLAS: the library DGEMMs of the wide-class fp64 path (csrc/snx_wide64.cu)
LINK = ["-lcublas", "-Xlinker", "-rpath", "-Xlinker", "/usr/local/cuda/lib64"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
         "--expt-relaxed-constexpr"]


def _nvcc():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libsnx")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + sorted(
        glob.glob(os.path.join(CSRC, "*.h"))) + sorted(glob.glob(os.path.join(INCLUDE, "*.h")))


def up_to_date():
    if not os.path.exists(LIBPATH):
        return False
    t = os.path.getmtime(LIBPATH)
    return all(os.path.getmtime(f) <= t for f in _deps())


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd))
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed ({proc.returncode}):\n{proc.stdout}\n{proc.stderr}")


def build(force=False, verbose=False):
    """Compile every csrc/*.cu for sm_100a (one object per source, rebuilt when
    it or a header changed; in parallel) and link _lib/libsnx.so."""
    if not force and up_to_date():
        return LIBPATH
    from concurrent.futures import ThreadPoolExecutor

    os.makedirs(OBJDIR, exist_ok=True)
    headers = [f for f in _deps() if not f.endswith(".cu")]
    newest_header = max(os.path.getmtime(f) for f in headers)
    compile_flags = [f for f in FLAGS if f != "-shared"]
    jobs, objs = [], []
    for src in sources():
        obj = os.path.join(OBJDIR, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(
                os.path.getmtime(src), newest_header):
            jobs.append([_nvcc(), *ARCH, *compile_flags, "-I", INCLUDE, "-c", src, "-o", obj])
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for f in [ex.submit(_run, cmd, verbose) for cmd in jobs]:
            f.result()
    os.makedirs(LIBDIR, exist_ok=True)
    tmp = LIBPATH + ".tmp"
    _run([_nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, *LINK, "-o", tmp], verbose)
    os.replace(tmp, LIBPATH)
    return LIBPATH


def build_timeline(out, extra=("-DSNX_TIMELINE",)):
    """Debug variant with per-CTA globaltimer stamps (tools/timeline.py with
    -DSNX_TIMELINE, tools/cl_timeline.py with -DSNX_CL_TIMELINE)."""
    cmd = [_nvcc(), *ARCH, *FLAGS, *extra, "-I", INCLUDE, *sources(), *LINK, "-o", out]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(proc.stderr)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=True))
