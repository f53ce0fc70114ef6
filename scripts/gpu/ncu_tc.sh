# ncu full capture (with SASS source counters) of coding_pass_tc on the c3s slice (tensor-core pass forced)
mkdir -p gpurun_out
export DCSC_TC=1
python bench.py --config c3s --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/n_c3s.json 2> gpurun_out/n_c3s.err || exit 1
ncu --set full --clock-control none --import-source on -k regex:coding_pass_tc -s 4 -c 1 -f -o gpurun_out/e_c3s_tc \
    python bench.py --config c3s --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/n_ncu.log 2>&1
ls -la gpurun_out
