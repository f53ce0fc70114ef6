# Round-2 (tensor-core pass) measurement batch (run under gpurun): bench lines,
# reference arm, ncu launch list and full captures of coding_pass_tc into gpurun_out/.
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 > gpurun_out/c_c3.json 2> gpurun_out/c_c3.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/c_c3_ref.json 2> gpurun_out/c_c3_ref.err
python bench.py --config c1 --steps 3 --warmup 3 > gpurun_out/c_c1.json 2> gpurun_out/c_c1.err
for c in c0 c2 c4; do python bench.py --config $c --steps 2 --warmup 3 > gpurun_out/c_${c}.json 2> gpurun_out/c_${c}.err; done
python bench.py --config c1j3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c_c1j3.json 2> gpurun_out/c_c1j3.err
python bench.py --config c3s --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c_c3s.json 2> gpurun_out/c_c3s.err
python scripts/family_times_run.py c3 3 > gpurun_out/c_c3_families.txt 2>&1
python bench.py --config c3s --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c_c3s_launches.csv \
    python bench.py --config c3s --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:coding_pass_tc -s 2 -c 1 -o gpurun_out/c_c3s_tc \
    python bench.py --config c3s --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c_ncu2.log 2>&1
python bench.py --config c1 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:coding_pass_tc -s 20 -c 1 -o gpurun_out/c_c1_tc \
    python bench.py --config c1 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c_ncu3.log 2>&1
echo done
