"""Build and run scripts/umma_probe.cu (tcgen05 layout / precision probe).

python scripts/umma_probe.py build   # here (nvcc cross-compiles)
python scripts/umma_probe.py run     # on the GPU box
"""
import ctypes
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(ROOT, "build", "umma_probe.so")


def build():
    os.makedirs(os.path.dirname(SO), exist_ok=True)
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
           "-I" + os.path.join(ROOT, "paper_1709_09479_b200", "csrc"),
           os.path.join(HERE, "umma_probe.cu"), "-o", SO]
    subprocess.check_call(cmd)


def run():
    lib = ctypes.CDLL(SO)
    f = ctypes.POINTER(ctypes.c_float)
    lib.umma_probe.argtypes = [f, f, f, ctypes.c_float, ctypes.c_float, f, f, ctypes.c_int]
    rng = np.random.default_rng(1)
    A1 = rng.standard_normal((128, 128)).astype(np.float32) * 3.0
    Dm = (rng.standard_normal((128, 128)) * 0.1).astype(np.float32)
    Dm[:, 121:] = 0
    Wm = (rng.standard_normal((128, 128)) * np.exp(rng.standard_normal((128, 1)) * 3)).astype(np.float32)
    sA = float(2.0 ** (14 - np.frexp(np.abs(A1).max())[1]))
    sD = float(2.0 ** (14 - np.frexp(np.abs(Dm).max())[1]))
    p = lambda a: a.ctypes.data_as(f)
    Tref = A1.astype(np.float64) @ Dm.astype(np.float64).T
    Zref = Wm.astype(np.float64) @ Dm.astype(np.float64)
    for variant in (0, 1):
        T = np.zeros((128, 128), np.float32)
        Z = np.zeros((128, 128), np.float32)
        rc = lib.umma_probe(p(A1), p(Dm), p(Wm), sA, sD, p(T), p(Z), variant)
        eT = np.abs(T - Tref).max() / np.abs(Tref).max()
        # Z rows have very different magnitudes: per-row relative error
        eZ = (np.abs(Z - Zref).max(axis=1) / np.maximum(np.abs(Zref).max(axis=1), 1e-30)).max()
        print(f"variant {variant} ({'3 products' if variant == 0 else 'hi*hi only'}): rc={rc} "
              f"T rel err {eT:.3e}  Z rel err (per row) {eZ:.3e}")
        if variant == 0 and not (eT < 1e-6 and eZ < 1e-6):
            # diagnose layout: correlation with permuted references
            print("T[0,:8]", T[0, :8]); print("Tref[0,:8]", Tref[0, :8])
            print("Z[0,:8]", Z[0, :8]); print("Zref[0,:8]", Zref[0, :8])
    out = (ctypes.c_longlong * 2)()
    lib.umma_time.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_longlong)]
    lib.umma_time(200, out)
    per = [out[i] / (200 * 24) for i in range(2)]
    print(f"cycles per 128x128x16 f16 MMA (A tmem): B K-major {per[0]:.1f}, B MN-major {per[1]:.1f}")
    # FP32 baseline error for comparison
    T32 = A1 @ Dm.T
    print("fp32 numpy T rel err", np.abs(T32 - Tref).max() / np.abs(Tref).max())


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]]()
