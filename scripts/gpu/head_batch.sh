# Bench lines of the other configs at HEAD (the default C3 line comes from head_check.sh).
mkdir -p gpurun_out
for c in c0 c1 c2 c4 c3s; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/h_${c}.json 2> gpurun_out/h_${c}.err; echo "$c rc=$?" >> gpurun_out/h_${c}.err
done
timeout 600 python scripts/fft_comparator.py > gpurun_out/h_fft_vs_cufft.jsonl 2> gpurun_out/h_fft.err; echo "fft rc=$?" >> gpurun_out/h_fft.err
for c in c0 c1 c2 c4 c3s; do python -c "
import json;d=json.loads(open('gpurun_out/h_${c}.json').read().strip().splitlines()[-1]);print('$c',round(d['value'],4),round(d['e2e']['value'],4),round(d['roofline']['frac'],3),d['clocks'])"; done
