# predicted W scale in the tensor-core pass: parity (tc, goldens at C1/C2/C3/C4, support), A/B vs the previous library
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -x tests/test_tc_gpu.py tests/test_golden_baseline_gpu.py tests/test_support_gpu.py tests/test_properties_gpu.py tests/test_golden_gpu.py > gpurun_out/w_tests.log 2>&1; echo "rc=$?" >> gpurun_out/w_tests.log
bash scripts/gpu/ab_cfg.sh c3m 3 prev > gpurun_out/w_ab.log 2>&1
bash scripts/gpu/ab_cfg.sh c1 3 prev >> gpurun_out/w_ab.log 2>&1
bash scripts/gpu/ab_cfg.sh c2 2 prev >> gpurun_out/w_ab.log 2>&1
