timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputest_full.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputest_full.log
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
