timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_grids_gpu.py tests/test_golden_gpu.py tests/test_golden_baseline_gpu.py > gpurun_out/t_fft.log 2>&1
timeout 300 python scripts/fft_comparator.py > gpurun_out/fft_cmp.jsonl 2> gpurun_out/fft_cmp.err
DCSC_NO_FFT_PIPE=1 timeout 300 python scripts/fft_comparator.py > gpurun_out/fft_cmp_nopipe.jsonl 2>> gpurun_out/fft_cmp.err
