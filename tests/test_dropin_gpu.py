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
