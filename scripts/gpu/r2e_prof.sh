# r02e evidence at HEAD: launch list and ncu full capture of coding_pass_tc on the c3s slice
# (tensor-core pass forced), a C1 capture, the C3 outer-iteration family breakdown, reference arm
mkdir -p gpurun_out
export DCSC_TC=1
python bench.py --config c3s --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e_c3s.json 2> gpurun_out/e_c3s.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/e_c3s_launches.csv \
    python bench.py --config c3s --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/e_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:coding_pass_tc -s 4 -c 1 -f -o gpurun_out/e_c3s_tc \
    python bench.py --config c3s --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/e_ncu2.log 2>&1
unset DCSC_TC
python bench.py --config c1 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:coding_pass_tc -s 20 -c 1 -f -o gpurun_out/e_c1_tc \
    python bench.py --config c1 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/e_ncu3.log 2>&1
python scripts/family_times_run.py c3 3 > gpurun_out/e_c3_families.txt 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/e_c3_ref.json 2> gpurun_out/e_c3_ref.err
ls -la gpurun_out | tail -20
