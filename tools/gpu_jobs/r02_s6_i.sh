mkdir -p gpurun_out
timeout 2000 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_s6i.json 2> gpurun_out/bench_s6i.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_s6i.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], 'clk', d['clocks'])
print(d['context'])"
tail -3 gpurun_out/bench_s6i.err
