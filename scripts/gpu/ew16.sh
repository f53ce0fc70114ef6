# 16 epilogue warps (two per group and TMEM lane quarter) vs 8: parity, then A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -x tests/test_tc_gpu.py tests/test_golden_baseline_gpu.py tests/test_support_gpu.py tests/test_golden_gpu.py > gpurun_out/w16_tests.log 2>&1; echo "rc=$?" >> gpurun_out/w16_tests.log
tail -5 gpurun_out/w16_tests.log
bash scripts/gpu/ab_cfg.sh c3m 3 ew8 > gpurun_out/w16_ab.log 2>&1
bash scripts/gpu/ab_cfg.sh c1 3 ew8 >> gpurun_out/w16_ab.log 2>&1
bash scripts/gpu/ab_cfg.sh c2 2 ew8 >> gpurun_out/w16_ab.log 2>&1
bash scripts/gpu/ab_cfg.sh c4 2 ew8 >> gpurun_out/w16_ab.log 2>&1
cat gpurun_out/w16_ab.log
