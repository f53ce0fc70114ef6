# round-2 measurement batch: every config's bench line + the reference arm (C3 default, C1)
for c in c1 c2 c4 c0 c1j3 c3s; do
  timeout 900 python bench.py --config $c > gpurun_out/r02_${c}_bench.json 2> gpurun_out/r02_${c}_bench.err
done
timeout 900 python bench.py --impl reference > gpurun_out/r02_c3_bench_reference_arm.json 2> gpurun_out/r02_ref_c3.err
timeout 900 python bench.py --impl reference --config c1 > gpurun_out/r02_c1_bench_reference_arm.json 2> gpurun_out/r02_ref_c1.err
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
