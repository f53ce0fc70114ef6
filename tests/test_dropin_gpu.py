"""GPU: a reference C++ program swaps dcsc::run_csc for dcsc::cuda::run_csc
(include/dcsc_cuda.hpp over the C-ABI) and gets the same trace (oracle/dropin_check.cpp)."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_check")


@pytest.mark.parametrize("channels", [1, 3])
def test_reference_program_drop_in(channels):
    if not os.path.exists(BIN):
        pytest.fail("oracle/_ref/dropin_check not built (make -C oracle dropin)")
    r = subprocess.run([BIN, "3", str(channels)], capture_output=True, text=True, timeout=300)
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert r.returncode == 0 and out["ok"], out


def test_reference_program_error_parity():
    """The drop-in throws the reference's exception type for the same bad input:
    empty / ragged datasets, non-finite signals, oversize support, no filters,
    negative beta (types.hpp:24-38, pipeline.cpp:66-80,159-167)."""
    if not os.path.exists(BIN):
        pytest.fail("oracle/_ref/dropin_check not built (make -C oracle dropin)")
    r = subprocess.run([BIN, "errors"], capture_output=True, text=True, timeout=300)
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert r.returncode == 0 and out["ok"], out
    assert len(out["errors"]) == 6


def test_reference_program_per_image_calls_from_openmp_threads():
    """The reference's per-image call pattern (pipeline.cpp:221-227): dcsc::cuda::solve_coding
    called concurrently from 4 OpenMP threads (each with its cached device context),
    warm states over two sweeps, then solve_learning; equal to the reference's
    sequential calls (iteration counts equal, maps <= 1e-9, dictionary <= 1e-7)."""
    if not os.path.exists(BIN):
        pytest.fail("oracle/_ref/dropin_check not built (make -C oracle dropin)")
    r = subprocess.run([BIN, "threads"], capture_output=True, text=True, timeout=300)
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert r.returncode == 0 and out["ok"], out


def test_run_csc_warnings_for_constant_inputs():
    """RunResult::warnings parity (pipeline.cpp:177-183): a constant image under
    Global normalisation is reported by name and mapped to zeros."""
    import numpy as np

    from paper_1709_09479_b200 import dcsc

    rng = np.random.default_rng(1)
    xs = rng.random((3, 16, 16))
    xs[1] = 0.25
    r = dcsc.run_csc(xs, 2, (3, 3), dcsc.SolverConfig(beta=0.2, max_outer=1, normalize=1, tol=1e-300), 64,
                     names=["a", "flat", "c"])
    assert r["warnings"] == ["normalize: constant input 'flat' mapped to zeros"]
