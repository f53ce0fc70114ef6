# HEAD validation: full GPU suite, smoke, default bench (C3), reference arm
mkdir -p gpurun_out
timeout 1700 python -m pytest tests -m gpu -q > gpurun_out/e_gputest.log 2>&1; echo "tests rc=$?" >> gpurun_out/e_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/e_smoke.log
timeout 900 python bench.py > gpurun_out/e_c3.json 2> gpurun_out/e_c3.err; echo "bench rc=$?" >> gpurun_out/e_gputest.log
timeout 600 python bench.py --impl reference > gpurun_out/e_c3_ref.json 2> gpurun_out/e_c3_ref.err; echo "ref rc=$?" >> gpurun_out/e_gputest.log
tail -3 gpurun_out/e_gputest.log
