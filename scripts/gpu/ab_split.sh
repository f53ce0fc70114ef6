# packed (main) vs scalar (var_sspl) f16 split in the tensor-core prox: parity tests on main, then A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_tc_gpu.py tests/test_support_gpu.py tests/test_golden_baseline_gpu.py -m gpu -x -q > gpurun_out/k_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/k_tests.log
tail -3 gpurun_out/k_tests.log
bash scripts/gpu/ab_cfg.sh c3 2 sspl 2>&1 | tee gpurun_out/k_ab_c3.log
for c in c1 c2 c4; do bash scripts/gpu/ab_cfg.sh $c 3 sspl 2>&1 | tee -a gpurun_out/k_ab_other.log; done
