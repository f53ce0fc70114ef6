DCSC_LIB=build/var_c0cl/libdcsc_cuda.so timeout 900 python -m pytest -q tests/test_golden_gpu.py tests/test_gpu_parity.py tests/test_properties_gpu.py -k "c0 or 100 or fp64" > gpurun_out/t_c0cl.log 2>&1
python scripts/ab.py c0 6 2 build/ab/head.so build/var_c0cl/libdcsc_cuda.so > gpurun_out/ab_c0cl.log 2>&1
