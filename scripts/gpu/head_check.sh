# HEAD verification: full GPU test suite, smoke, the driver's default bench line and the reference arm.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/f_gputest.log 2>&1; echo "tests rc=$?" >> gpurun_out/f_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f_smoke.log
timeout 900 python bench.py > gpurun_out/f_c3.json 2> gpurun_out/f_c3.err; echo "bench rc=$?" >> gpurun_out/f_c3.err
timeout 900 python bench.py --impl reference > gpurun_out/f_c3_ref.json 2> gpurun_out/f_c3_ref.err; echo "ref rc=$?" >> gpurun_out/f_c3_ref.err
tail -3 gpurun_out/f_gputest.log; tail -2 gpurun_out/f_smoke.log; cat gpurun_out/f_c3.json
