# One ncu --set full capture of a full-size C3 half-batch coding_pass_tc launch (256 images) from the default bench command.
mkdir -p gpurun_out
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:coding_pass_tc -s 3500 -c 1 -o gpurun_out/i_c3_tc -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/i_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/i_ncu.log
tail -3 gpurun_out/i_ncu.log | cut -c1-400; ls -la gpurun_out/i_c3_tc.ncu-rep
