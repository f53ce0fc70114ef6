"""CPU: the C-ABI library loads and exports every symbol include/dcsc_cuda.h
declares; argument validation and the data generator (no GPU compute)."""
import os
import re

import numpy as np
import pytest

from paper_1709_09479_b200 import dcsc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dcsc_cuda.h")).read()
    return sorted(set(re.findall(r"\bint\s+(dcsc_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = dcsc.lib()
    syms = declared_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(dcsc.EXPORTS)


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", dcsc.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_supported_grids():
    assert dcsc.supported_grid(128, 128, 32)
    assert dcsc.supported_grid(100, 100, 64)
    assert not dcsc.supported_grid(127, 128, 32)


def test_invalid_config_is_rejected_before_device_work():
    with pytest.raises(dcsc.InvalidArgument):
        dcsc.Context(1, (16, 16), 2, (3, 3), dcsc.SolverConfig(beta=-1.0))
    with pytest.raises(dcsc.InvalidArgument):
        dcsc.Context(1, (16, 16), 2, (3, 3), dcsc.SolverConfig(cg_max=0))
    with pytest.raises(dcsc.DimensionError):
        dcsc.Context(1, (16, 16), 2, (17, 3), dcsc.SolverConfig())
    with pytest.raises(dcsc.DimensionError):
        dcsc.Context(1, (18, 18), 2, (3, 3), dcsc.SolverConfig())


def test_synth_is_deterministic_and_shaped():
    x1, d1 = dcsc.synth_generate(3, (20, 20), 4, 5, 0.05, 0.01, 11, False)
    x2, d2 = dcsc.synth_generate(3, (20, 20), 4, 5, 0.05, 0.01, 11, False)
    assert np.array_equal(x1, x2) and np.array_equal(d1, d2)
    assert np.allclose(np.sqrt((d1 ** 2).sum(axis=(1, 2))), 1.0)
    assert np.abs(x1.mean(axis=(1, 2))).max() < 1e-12
    x3, _ = dcsc.synth_generate(3, (20, 20), 4, 5, 0.05, 0.01, 12, False)
    assert not np.array_equal(x1, x3)


def test_synth_fp32_rounding():
    x, _ = dcsc.synth_generate(2, (16, 16), 2, 3, 0.1, 0.01, 1, True)
    assert np.array_equal(x, x.astype(np.float32).astype(np.float64))


def test_synth_images_independent_of_batch():
    # image n's stream depends only on (seed, n): a rank can generate its shard alone
    xa, _ = dcsc.synth_generate(4, (16, 16), 2, 3, 0.1, 0.01, 5, False)
    xb, _ = dcsc.synth_generate(2, (16, 16), 2, 3, 0.1, 0.01, 5, False)
    assert np.array_equal(xa[:2], xb)


def test_channel_count_is_validated_before_touching_the_device():
    # J > 8 is rejected by the engine constructor (DimensionError) on any host
    with pytest.raises(dcsc.DimensionError):
        dcsc.Context(2, (20, 20), 4, (5, 5), dcsc.SolverConfig(normalize=0), 64, channels=9)


def test_cluster_grid_limits_are_dimension_errors():
    # the 4-CTA cluster families crop the support inside rank 0's row block
    # (H / 4 rows) and every family takes at most 8 channels: checked before
    # any device work, so this runs without a GPU
    with pytest.raises(dcsc.DimensionError):
        dcsc.Context(1, (256, 256), 4, (65, 65), dcsc.SolverConfig(normalize=0), 32)
    with pytest.raises(dcsc.DimensionError):
        dcsc.Context(1, (128, 128), 4, (33, 5), dcsc.SolverConfig(normalize=0), 64)
    with pytest.raises(dcsc.DimensionError):
        dcsc.Context(1, (64, 64), 4, (5, 5), dcsc.SolverConfig(normalize=0), 32, channels=9)
