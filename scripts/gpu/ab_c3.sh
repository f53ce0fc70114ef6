# C3 headline A/B (full bench default: outers 4-6) between the main library and variants
for r in 1 2; do
  for lib in main "$@"; do
    if [ "$lib" = main ]; then unset DCSC_LIB; else export DCSC_LIB=build/var_$lib/libdcsc_cuda.so; fi
    timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/abc3.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/abc3.json').read().strip().splitlines()[-1]);print('c3 $lib', round(d['value'],5), round(d['roofline']['coding_phase_ms'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
