# A/B of coding_pass_tc variants on c3s (DCSC_TC=1): ms per launch, alternating libraries
export DCSC_TC=1
for r in 1 2; do
  for lib in main "$@"; do
    if [ "$lib" = main ]; then unset DCSC_LIB; else export DCSC_LIB=build/var_$lib/libdcsc_cuda.so; fi
    timeout 300 python bench.py --config c3s --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$lib', round(d['roofline']['avg_launch_ms'],4))"
  done
done
