# A/B of library variants on one bench config: CONFIG STEPS variant-tags...; prints the
# coding-pass ms per launch and the step value of each run, alternating libraries
cfg=$1; steps=$2; shift 2
for r in 1 2; do
  for lib in main "$@"; do
    if [ "$lib" = main ]; then unset DCSC_LIB; else export DCSC_LIB=build/var_$lib/libdcsc_cuda.so; fi
    timeout 600 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$cfg $lib', round(d['roofline']['avg_launch_ms'],4), round(d['value'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
