mkdir -p gpurun_out
cp paper_2601_11437_b200/libmaternfisher.so /tmp/lib_default.so
for v in serial default; do
  if [ $v = default ]; then cp /tmp/lib_default.so paper_2601_11437_b200/libmaternfisher.so; else cp gpurun_variants/lib_$v.so paper_2601_11437_b200/libmaternfisher.so; fi
  timeout 600 python tools/stage_ab.py --child 2>&1 | grep RESULT > gpurun_out/diag_ab_$v.json
  timeout 300 python tools/diag_trace_probe.py > gpurun_out/diag_trace_$v.txt 2>&1
done
cp /tmp/lib_default.so paper_2601_11437_b200/libmaternfisher.so
python - <<'PY'
import json
r={v:json.loads(open(f'gpurun_out/diag_ab_{v}.json').read()[7:]) for v in ('serial','default')}
for k in ('config2_bits','config3_bits'): print(k,'equal',r['serial'][k]==r['default'][k])
for v in r: print(v,{k:(round(x,3) if isinstance(x,float) else x) for k,x in r[v].items() if k.endswith('_ms')}, 'potrf', r[v]['config2_batched_loglik_phases']['potrf_ms'], 'c3 potrf', r[v]['config3_phases']['potrf_ms'])
PY
head -12 gpurun_out/diag_trace_serial.txt; head -12 gpurun_out/diag_trace_default.txt
