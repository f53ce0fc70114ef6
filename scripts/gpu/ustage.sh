timeout 900 python -m pytest -q -x tests/test_golden_baseline_gpu.py tests/test_support_gpu.py tests/test_gpu_parity.py tests/test_dropin_gpu.py -k "cluster or c3 or support or 256 or dropin or reference_program or warnings" > gpurun_out/t_cl.log 2>&1
python scripts/ab.py c3s 60 2 main build/var_nou/libdcsc_cuda.so > gpurun_out/ab.log 2>&1
DCSC_LIB=build/var_trace/libdcsc_cuda.so timeout 300 python bench.py --config c3s --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/c3s_trace.json 2> gpurun_out/c3s_trace.err
