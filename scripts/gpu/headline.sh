timeout 900 python bench.py > gpurun_out/r02_c3_bench.json 2> gpurun_out/r02_c3_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r02_c3_bench_reference_arm.json 2> gpurun_out/r02_ref_c3.err
timeout 600 python bench.py --config c3s --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02_c3s_bench.json 2> gpurun_out/r02_c3s_bench.err
