mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s7j.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke_s7j.log | cut -c 1-120
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputest_s7j.log 2>&1; echo gputest rc=$?; tail -2 gpurun_out/gputest_s7j.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_s7j.json 2> gpurun_out/bench_s7j.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_s7j.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], 'clk', d['clocks'])
k=d['kernels']; print({x:k.get(x) for x in ('ozgemm_alg_fp64_equiv_tflops','eval_all_ms','gen_gbs','gen_ms')}); print(k.get('generation_ncu'))"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_s7j.json 2>/dev/null; echo ref rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_s7j.csv python tools/prof_config4.py > /dev/null 2>&1; echo launches rc=$?
python tools/launch_summary.py gpurun_out/launches_c4_s7j.csv > gpurun_out/launches_c4_s7j_summary.txt; head -10 gpurun_out/launches_c4_s7j_summary.txt
for s in 1; do MLE_GEN_STAGE=$s timeout 600 python tools/gen_config4_probe.py config4 2>&1 | grep GENPROBE > gpurun_out/gen_probe_c4_final.json; done
python - <<'PY'
import json
base=json.loads(open('tools/gen_probe_c4_baseline_bits.json').read()[9:])
r=json.loads(open('gpurun_out/gen_probe_c4_final.json').read()[9:])
print('config-4 bits equal to the session-start build:', r['bits']==base['bits'], {k:round(v,1) for k,v in r.items() if k not in ('bits','workload')})
PY
