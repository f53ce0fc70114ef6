"""In-tree build of the sm_100a library paper_1709_09479_b200/lib/libdcsc_cuda.so.

nvcc cross-compiles for sm_100a on a machine without a GPU; the built .so is
git-ignored but travels with the gpurun snapshot. Object files are cached in
build/ and rebuilt only when a source or header is newer.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
LIBDIR = os.path.join(PKG, "lib")
OBJDIR = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(LIBDIR, "libdcsc_cuda.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-fopenmp", "-Xptxas", "-v", "-I" + INC, "-I" + CSRC,
]
HOST_CXX = shutil.which("g++", path="/usr/bin") or "g++"


def _nvcc() -> str:
    for p in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if p and os.path.exists(p):
            return p
    raise RuntimeError("nvcc not found")


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h", ".hpp"))]
    hs += [os.path.join(INC, f) for f in os.listdir(INC)]
    return hs


def _stale(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, defines=(), tag=None, only=None) -> str:
    """Build the library. Experiment variants: `tag` builds build/var_<tag>/libdcsc_cuda.so
    with extra -D `defines`, recompiling only the units named in `only` (the
    rest are the default objects); load it with DCSC_LIB=<path>."""
    lib, objdir = LIB, OBJDIR
    if tag:
        lib = os.path.join(ROOT, "build", "var_" + tag, "libdcsc_cuda.so")
        objdir = os.path.join(ROOT, "build", "obj_" + tag)
        build()
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    os.makedirs(objdir, exist_ok=True)
    nvcc = _nvcc()
    hdrs = _headers()
    objs, jobs = [], []
    for src in sorted(os.listdir(CSRC)):
        path = os.path.join(CSRC, src)
        if not src.endswith((".cu", ".cpp")):
            continue
        if tag and src not in (only or ()):
            objs.append(os.path.join(OBJDIR, src + ".o"))
            continue
        obj = os.path.join(objdir, src + ".o")
        objs.append(obj)
        if not _stale(obj, [path] + hdrs) and not tag:
            continue
        if src.endswith(".cu"):
            cmd = [nvcc, "-c", path, "-o", obj] + NVCC_FLAGS + ["-D" + d for d in defines] + ["-ccbin", HOST_CXX]
        else:
            cmd = [HOST_CXX, "-c", path, "-o", obj, "-O3", "-fPIC", "-fopenmp", "-std=c++17", "-I" + INC, "-I" + CSRC]
        jobs.append((src, cmd))

    def run(job):
        src, cmd = job
        log = os.path.join(objdir, src + ".build.log")
        with open(log, "w") as f:
            r = subprocess.run(cmd, stdout=f, stderr=subprocess.STDOUT)
        return src, r.returncode, log

    # the per-grid engine units (inst_*.cu) are independent: compile in parallel
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for src, rc, log in ex.map(run, jobs):
            if rc != 0:
                sys.stderr.write(open(log).read()[-20000:])
                raise RuntimeError(f"compile failed on {src}")
    if _stale(lib, objs) or tag:
        cmd = [nvcc, "-shared", "-o", lib] + objs + ARCH + ["-ccbin", HOST_CXX, "-Xcompiler", "-fopenmp", "-lgomp"]
        subprocess.run(cmd, check=True)
    return lib


GRIDDIR = os.path.join(LIBDIR, "grids")


def _smooth(n: int) -> bool:
    for p in (2, 3, 5):
        while n % p == 0:
            n //= p
    return n == 1


def grid_lib(precision: int, H: int, W: int) -> str:
    return os.path.join(GRIDDIR, f"libdcsc_grid_f{precision}_{H}x{W}.so")


def build_grid(precision: int, H: int, W: int, force: bool = False) -> str:
    """Compile the engine for one more grid as a plugin library (DCSC_GRID_PLUGIN,
    csrc/engine_impl.cuh): lib/grids/libdcsc_grid_f<P>_<H>x<W>.so, which the main library
    finds by name (the reference plans any grid at run time, spectral.cpp:16-47; here a
    grid is a compiled kernel family). One CTA holds a half-spectrum plane in shared
    memory, so H x (W/2 + 1) complex values must fit; H and W/2 must factor into 2, 3, 5."""
    if precision not in (32, 64):
        raise ValueError("precision must be 32 or 64")
    if H < 8 or W < 16 or W % 2 or not _smooth(H) or not _smooth(W // 2):
        raise ValueError(f"grid {H}x{W}: W must be even, H >= 8, W >= 16, and H, W/2 must factor into 2, 3 and 5")
    plane = H * (W // 2 + 1) * (8 if precision == 32 else 16)
    limit = 66560 if precision == 32 else 81600  # the largest single-CTA families: FP32 128x128, FP64 100x100
    if plane > limit:
        raise ValueError(f"grid {H}x{W} FP{precision}: half-spectrum plane of {plane} bytes exceeds the "
                         f"single-CTA family's {limit}")
    lib = grid_lib(precision, H, W)
    hdrs = _headers()
    if not force and not _stale(lib, hdrs):
        return lib
    os.makedirs(GRIDDIR, exist_ok=True)
    gdir = os.path.join(ROOT, "build", "grids")
    os.makedirs(gdir, exist_ok=True)
    rt = "float" if precision == 32 else "double"
    src = os.path.join(gdir, f"grid_f{precision}_{H}x{W}.cu")
    with open(src, "w") as f:
        f.write(f"// generated by build.build_grid: engine plugin for {rt} {H}x{W}\n"
                f'#include "engine_impl.cuh"\n\nDCSC_GRID_PLUGIN({rt}, {H}, {W})\n')
    log = src + ".build.log"
    cmd = [_nvcc(), "-shared", src, "-o", lib] + NVCC_FLAGS + ["-ccbin", HOST_CXX, "-lgomp"]
    with open(log, "w") as f:
        r = subprocess.run(cmd, stdout=f, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        sys.stderr.write(open(log).read()[-20000:])
        raise RuntimeError(f"grid plugin {rt} {H}x{W} failed to compile")
    return lib


if __name__ == "__main__":
    if len(sys.argv) >= 5 and sys.argv[1] == "--grid":
        print(build_grid(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])))
    else:
        print(build(verbose=True))
