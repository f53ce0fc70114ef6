# GEMM-2 K-steps pipelined behind the prox (Z into the im2col half): parity, then A/B vs the previous library
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -x tests/test_tc_gpu.py tests/test_golden_baseline_gpu.py tests/test_support_gpu.py > gpurun_out/p_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p_tests.log
tail -3 gpurun_out/p_tests.log
bash scripts/gpu/ab_cfg.sh c3m 3 prev > gpurun_out/p_ab.log 2>&1
bash scripts/gpu/ab_cfg.sh c1 3 prev >> gpurun_out/p_ab.log 2>&1
bash scripts/gpu/ab_cfg.sh c2 2 prev >> gpurun_out/p_ab.log 2>&1
bash scripts/gpu/ab_cfg.sh c4 2 prev >> gpurun_out/p_ab.log 2>&1
cat gpurun_out/p_ab.log
