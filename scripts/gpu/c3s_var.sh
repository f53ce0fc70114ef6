for v in main s1 l1; do
  if [ $v = main ]; then L=""; else L="DCSC_LIB=build/var_$v/libdcsc_cuda.so"; fi
  env $L timeout 300 python bench.py --config c3s --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c3s_$v.json 2> gpurun_out/c3s_$v.err
done
DCSC_LIB=build/var_trace/libdcsc_cuda.so timeout 300 python bench.py --config c3s --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/c3s_trace.json 2> gpurun_out/c3s_trace.err
