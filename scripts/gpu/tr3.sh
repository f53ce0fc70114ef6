mkdir -p gpurun_out
for v in trace_prev trace trace_pipe1; do
DCSC_TC=1 DCSC_LIB=build/var_$v/libdcsc_cuda.so timeout 300 python bench.py --config c3s --steps 1 --warmup 1 --no-cpu-baseline 2> gpurun_out/tr_$v.err | grep TCT | head -12 > gpurun_out/tr_$v.txt
echo $v; cat gpurun_out/tr_$v.txt
done
