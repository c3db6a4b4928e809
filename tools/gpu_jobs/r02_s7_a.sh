mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s7b.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke_s7b.log | cut -c 1-200
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gputest_s7b.log 2>&1; echo gputest rc=$?; tail -25 gpurun_out/gputest_s7b.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_s7b.json 2> gpurun_out/bench_s7b.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_s7b.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], 'achieved', d['roofline']['achieved'], 'clk', d['clocks'])
k=d['kernels']; print({x:k.get(x) for x in ('ozgemm_alg_fp64_equiv_tflops','solve_path','eval_all_ms','reference_equivalent_tflops','gen_gbs','gen_ms')}); print(d['context'])"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_s7b.json 2>/dev/null; echo ref rc=$?; tail -c 600 gpurun_out/bench_ref_s7b.json
