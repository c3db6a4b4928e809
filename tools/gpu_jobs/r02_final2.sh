mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_f2.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke_f2.log | cut -c 1-200
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputest_f2.log 2>&1; echo gputest rc=$?; tail -3 gpurun_out/gputest_f2.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_f2.json 2> gpurun_out/bench_f2.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_f2.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], 'achieved', d['roofline']['achieved'], 'traffic', d['roofline']['traffic'], 'clk', d['clocks'])
k=d['kernels']; print({x:k.get(x) for x in ('ozgemm_alg_fp64_equiv_tflops','solve_path','eval_all_ms','reference_equivalent_tflops','gen_gbs')}); print(d['context']); print(d.get('cpu_baseline'))"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_f2.json 2>/dev/null; echo ref rc=$?; python -c "
import json; d=json.loads(open('gpurun_out/bench_ref_f2.json').read().strip().splitlines()[-1]); print('ref value', d['value'], d['cpu_baseline']['cores'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_final.csv python tools/prof_config4.py > /dev/null 2>&1; echo launches rc=$?
python tools/launch_summary.py gpurun_out/launches_c4_final.csv > gpurun_out/launches_c4_final_summary.txt; head -8 gpurun_out/launches_c4_final_summary.txt
