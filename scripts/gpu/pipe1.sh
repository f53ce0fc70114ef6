mkdir -p gpurun_out
for v in trace_prev trace trace_pipe1; do
DCSC_TC=1 DCSC_LIB=build/var_$v/libdcsc_cuda.so timeout 300 python bench.py --config c3s --steps 1 --warmup 1 --no-cpu-baseline 2> gpurun_out/tr_$v.err | grep TCT | head -12 > gpurun_out/tr_$v.txt
done
DCSC_LIB=build/var_pipe1/libdcsc_cuda.so timeout 600 python -m pytest -q -x tests/test_tc_gpu.py tests/test_support_gpu.py > gpurun_out/p1_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p1_tests.log
bash scripts/gpu/ab_cfg.sh c3m 3 prev pipe1 > gpurun_out/p1_ab.log 2>&1
bash scripts/gpu/ab_cfg.sh c1 3 prev pipe1 >> gpurun_out/p1_ab.log 2>&1
cat gpurun_out/p1_ab.log; tail -2 gpurun_out/p1_tests.log; cat gpurun_out/tr_*.txt
