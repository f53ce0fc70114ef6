# bench lines after the two-stream default and KF = 112 (C1, C2, C4, C3)
mkdir -p gpurun_out
python bench.py --config c1 --steps 3 --warmup 3 > gpurun_out/d_c1.json 2> gpurun_out/d_c1.err
for c in c2 c4; do python bench.py --config $c --steps 2 --warmup 3 > gpurun_out/d_${c}.json 2> gpurun_out/d_${c}.err; done
python bench.py --steps 3 --warmup 3 > gpurun_out/d_c3.json 2> gpurun_out/d_c3.err
echo done
