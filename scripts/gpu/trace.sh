DCSC_LIB=build/var_trace/libdcsc_cuda.so timeout 300 python bench.py --config c3s --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/c3s_trace.json 2> gpurun_out/c3s_trace.err
