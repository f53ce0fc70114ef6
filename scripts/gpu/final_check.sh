timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputest_full.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputest_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
