# plain runs first (exit 0), then ncu: C3 headline launch list, the C3 cluster coding pass (c3s), the
# C1 coding pass, the pipelined 128^2 r2c
set -e
python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/plain_c3.log 2>&1
python bench.py --config c3s --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_c3s.log 2>&1
python bench.py --config c1 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_c1.log 2>&1
python scripts/fft_comparator.py > gpurun_out/plain_fft.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/r02_c3_launches.csv python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_c3_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:coding_pass_cl -s 6 -c 1 -o gpurun_out/r02_c3s_cl -f python bench.py --config c3s --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c3s.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:coding_pass -s 8 -c 1 -o gpurun_out/r02_c1_cp -f python bench.py --config c1 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c1.log 2>&1
ncu --set full --clock-control none -k regex:r2c_planes_pipe -s 3 -c 1 -o gpurun_out/r02_r2c_pipe -f python scripts/fft_comparator.py > gpurun_out/ncu_fft.log 2>&1
