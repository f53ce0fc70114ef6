timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputest_full.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputest_full.log
DCSC_BENCH_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config c4 --learning-layout freq --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c4_gloo2_freq.json 2> gpurun_out/bench_c4_gloo2_freq.err; echo "gloo rc=$?" >> gpurun_out/gputest_full.log
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
