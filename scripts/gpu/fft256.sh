timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_golden_baseline_gpu.py -k "256 or cluster or c3 or dft" > gpurun_out/t_fft256.log 2>&1
timeout 300 python scripts/fft_comparator.py > gpurun_out/fft_cmp.jsonl 2> gpurun_out/fft_cmp.err
