mkdir -p gpurun_out
python tools/stage_ab.py MLE_GEN_STAGE=0 MLE_GEN_STAGE=1 > gpurun_out/gen_stage_ab.txt 2>&1; cat gpurun_out/gen_stage_ab.txt | cut -c 1-900
for s in 0 1; do MLE_GEN_STAGE=$s timeout 600 python tools/gen_config4_probe.py config4 2>&1 | grep GENPROBE > gpurun_out/gen_probe_c4_stage$s.json; done
python - <<'PY'
import json
r=[json.loads(open(f'gpurun_out/gen_probe_c4_stage{s}.json').read()[9:]) for s in (0,1)]
print('bits equal', r[0]['bits']==r[1]['bits'])
for x in r: print({k:v for k,v in x.items() if k!='bits'})
PY
MLE_GEN_STAGE=1 python tools/gen_bench.py 2>&1 | grep "gen GB" | tail -2
MLE_GEN_STAGE=0 python tools/gen_bench.py 2>&1 | grep "gen GB" | tail -2
