mkdir -p gpurun_out
DCSC_LIB=build/var_sgen/libdcsc_cuda.so python scripts/bitcheck_tc.py write /tmp/bit_ref.npz 2>&1 | tail -1
python scripts/bitcheck_tc.py compare /tmp/bit_ref.npz 2>&1 | tail -1
timeout 900 python -m pytest tests/test_tc_gpu.py tests/test_support_gpu.py tests/test_golden_baseline_gpu.py -m gpu -x -q 2>&1 | tail -2
bash scripts/gpu/ab_cfg.sh c3 2 sgen 2>&1 | tee gpurun_out/m_ab_strip.log
