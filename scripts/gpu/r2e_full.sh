# full GPU suite + smoke + bench lines of every config at HEAD (r02e)
mkdir -p gpurun_out
timeout 1700 python -m pytest tests -m gpu -q > gpurun_out/e_gputest.log 2>&1; echo "tests rc=$?" >> gpurun_out/e_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/e_smoke.log
timeout 900 python bench.py > gpurun_out/e_c3.json 2> gpurun_out/e_c3.err; echo "bench rc=$?" >> gpurun_out/e_gputest.log
python bench.py --config c1 --steps 3 --warmup 3 > gpurun_out/e_c1.json 2> gpurun_out/e_c1.err
for c in c0 c2 c4; do python bench.py --config $c --steps 2 --warmup 3 > gpurun_out/e_${c}.json 2> gpurun_out/e_${c}.err; done
tail -3 gpurun_out/e_gputest.log; tail -2 gpurun_out/e_smoke.log
for c in c3 c1 c0 c2 c4; do python -c "import json;d=json.loads(open('gpurun_out/e_$c.json').read().strip().splitlines()[-1]);print('$c', round(d['value'],4), d['e2e']['value'], d['roofline']['frac'], d['clocks'])"; done
