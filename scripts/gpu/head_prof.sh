# New edge tests, then the ncu launch list of the driver's default bench command (C3, tensor-core path).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_edge_gpu.py -m gpu -q > gpurun_out/g_edge.log 2>&1; echo "edge rc=$?" >> gpurun_out/g_edge.log
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g_c3_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/g_ncu_c3.log 2>&1; echo "ncu rc=$?" >> gpurun_out/g_ncu_c3.log
tail -15 gpurun_out/g_edge.log
