mkdir -p gpurun_out
for s in 0 1; do MLE_GEN_STAGE=$s timeout 600 python tools/gen_config4_probe.py config4 2>&1 | grep GENPROBE > gpurun_out/gen_probe_c4_v2_stage$s.json; done
python - <<'PY'
import json
base=json.loads(open('tools/gen_probe_c4_baseline_bits.json').read()[9:])
r=[json.loads(open(f'gpurun_out/gen_probe_c4_v2_stage{s}.json').read()[9:]) for s in (0,1)]
print('bits equal to the pre-change build:', [x['bits']==base['bits'] for x in r])
print('baseline', {k:v for k,v in base.items() if k!='bits'})
for x in r: print({k:v for k,v in x.items() if k!='bits'})
PY
MLE_GEN_STAGE=1 python tools/gen_bench.py 2>&1 | grep "gen GB" | tail -1
MLE_GEN_STAGE=0 python tools/gen_bench.py 2>&1 | grep "gen GB" | tail -1
timeout 900 python -m pytest tests/test_gpu_likelihood.py tests/test_gpu_special.py tests/test_gpu_fits.py tests/test_gpu_nugget.py -m gpu -x -q 2>&1 | tail -3
