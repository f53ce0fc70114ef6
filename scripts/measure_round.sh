# Round-end measurement batch (run under gpurun): bench lines, traces, ncu launch list and full captures into gpurun_out/.
mkdir -p gpurun_out
python bench.py > gpurun_out/m_c1.json 2> gpurun_out/m_c1.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/m_c1_ref.json 2>&1
for c in c0 c2 c4; do python bench.py --config $c --steps 2 --warmup 2 > gpurun_out/m_${c}.json 2> gpurun_out/m_${c}.err; done
python bench.py --config c1j3 --steps 3 --warmup 3 > gpurun_out/m_c1j3.json 2> gpurun_out/m_c1j3.err
python bench.py --config c3s --steps 5 --warmup 3 > gpurun_out/m_c3s.json 2> gpurun_out/m_c3s.err
python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/m_c3.json 2> gpurun_out/m_c3.err
python scripts/run_trace.py c2 2 > gpurun_out/m_c2_trace.json 2>/dev/null
python scripts/run_trace.py c4 2 > gpurun_out/m_c4_trace.json 2>/dev/null
python scripts/run_trace.py c3 1 > gpurun_out/m_c3_trace.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/m_c1_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/m_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:coding_pass -s 20 -c 1 -o gpurun_out/m_c1_cp python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/m_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:coding_pass_cl -s 5 -c 1 -o gpurun_out/m_c3s_cl python bench.py --config c3s --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/m_ncu3.log 2>&1
echo done
