timeout 300 python bench.py --config c3s --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c3s_new.json 2> gpurun_out/c3s_new.err
DCSC_LIB=build/var_trace/libdcsc_cuda.so timeout 300 python bench.py --config c3s --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/c3s_trace.json 2> gpurun_out/c3s_trace.err
timeout 600 python -m pytest -q -x tests/test_golden_baseline_gpu.py tests/test_support_gpu.py tests/test_gpu_parity.py -k "cluster or c3 or support or 256" > gpurun_out/t_cl.log 2>&1
echo done
