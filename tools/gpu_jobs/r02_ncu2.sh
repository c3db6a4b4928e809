# ncu of the current build at config 4: launch list of one Fisher iteration, --set full of the
# largest Ozaki GEMM launch and of the derivative-generation launch.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_v2.csv python tools/prof_config4.py > gpurun_out/launches_c4_v2.log 2>&1; echo launches rc=$?
python tools/launch_summary.py gpurun_out/launches_c4_v2.csv > gpurun_out/launches_c4_v2_summary.txt 2>&1; head -14 gpurun_out/launches_c4_v2_summary.txt
python - <<'PY' > gpurun_out/oz_idx.txt
import csv
rows=[r for r in csv.reader(open('gpurun_out/launches_c4_v2.csv')) if r]
hdr=next(r for r in rows if r[0]=='ID'); data=[dict(zip(hdr,r)) for r in rows if len(r)==len(hdr) and r[0]!='ID']
oz=[d for d in data if 'ozgemm_persistent' in d['Kernel Name']]
best=max(range(len(oz)), key=lambda i: float(oz[i]['Metric Value']))
print(best, oz[best]['Metric Value'])
PY
IDX=$(cut -d' ' -f1 gpurun_out/oz_idx.txt); echo "largest ozgemm launch: $(cat gpurun_out/oz_idx.txt)"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ozgemm_persistent --launch-skip $IDX -c 1 -o gpurun_out/r02_ozgemm_config4_v2 python tools/prof_config4.py > gpurun_out/ncu_full_v2.log 2>&1; echo ncu oz rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_engine_kernel -c 3 -o gpurun_out/r02_gen_config4 python tools/prof_config4.py > gpurun_out/ncu_gen.log 2>&1; echo ncu gen rc=$?
python tools/ncu_summary.py gpurun_out/r02_ozgemm_config4_v2.ncu-rep gpurun_out/r02_gen_config4.ncu-rep > gpurun_out/r02_ncu_config4_summary.txt 2>&1; cat gpurun_out/r02_ncu_config4_summary.txt
