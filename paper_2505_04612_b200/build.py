"""Build the C-ABI shared library ``libfastmap_b200.so`` in-tree for sm_100a.

Plain ``nvcc`` (no torch extension machinery): the library exports the
``extern "C"`` functions declared in ``include/fastmap_b200.h`` and links the
CUDA runtime statically, so it loads on a CPU-only host (the driver is only
touched by the first CUDA call).
"""

import os
import shutil
import subprocess
import sys

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
CSRC = os.path.join(PKG_DIR, "csrc")
LIB_NAME = "libfastmap_b200.so"
LIB_PATH = os.path.join(PKG_DIR, LIB_NAME)
SOURCES = ["fm_core.cu", "fm_store.cu", "fm_point_pass.cu", "fm_epipolar.cu", "fm_translation.cu", "fm_sphere.cu",
           "fm_fundamental.cu", "fm_rotation.cu", "fm_tracks.cu", "fm_dist.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale():
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(REPO_DIR, "include", "fastmap_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, extra=(), out=None):
    """Compile every CUDA source into LIB_PATH (skipped when up to date).
    The translation units compile in parallel (one nvcc per source), then
    link into one shared library."""
    if out is None and not force and not _stale():
        return LIB_PATH
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    target = out or LIB_PATH
    tmp = target + ".tmp"
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "--extended-lambda", "-Xcompiler", "-fPIC",
             "-I", os.path.join(REPO_DIR, "include"), *extra]
    with tempfile.TemporaryDirectory() as td:
        objs = [os.path.join(td, s.replace(".cu", ".o")) for s in SOURCES]
        cmds = [[nvcc_path(), *flags, "-c", os.path.join(CSRC, s), "-o", o]
                for s, o in zip(SOURCES, objs)]
        if verbose:
            for c in cmds:
                print(" ".join(c), file=sys.stderr)
        with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as ex:
            procs = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), cmds))
        for c, p in zip(cmds, procs):
            sys.stderr.write(p.stderr)
            if p.returncode:
                raise subprocess.CalledProcessError(p.returncode, c)
        subprocess.run([nvcc_path(), *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs],
                       check=True)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True,
          extra=["-Xptxas", "-v"] if "--ptxas" in sys.argv else [])
    print(LIB_PATH)
