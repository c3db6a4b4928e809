# Round-2 full cycle: GPU tests, bench (config 4), ncu launch list of one config-4 Fisher
# iteration, ncu --set full of its largest Ozaki GEMM launch.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputest_full.log 2>&1; echo gputest rc=$?; tail -4 gpurun_out/gputest_full.log
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench rc=$?
tail -c 600 gpurun_out/bench_c4.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python tools/prof_config4.py > gpurun_out/launches_c4.log 2>&1; echo launches rc=$?
python tools/launch_summary.py gpurun_out/launches_c4.csv > gpurun_out/launches_c4_summary.txt 2>&1; head -20 gpurun_out/launches_c4_summary.txt
python - <<'PY' > gpurun_out/oz_idx.txt
import csv
rows=[r for r in csv.reader(open('gpurun_out/launches_c4.csv')) if r]
hdr=next(r for r in rows if r[0]=='ID'); data=[dict(zip(hdr,r)) for r in rows if len(r)==len(hdr) and r[0]!='ID']
oz=[d for d in data if 'ozgemm_persistent' in d['Kernel Name']]
best=max(range(len(oz)), key=lambda i: float(oz[i]['Metric Value']))
print(best, oz[best]['Metric Value'])
PY
IDX=$(cut -d' ' -f1 gpurun_out/oz_idx.txt); echo "largest ozgemm launch $IDX: $(cat gpurun_out/oz_idx.txt)"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ozgemm_persistent --launch-skip $IDX -c 1 -o gpurun_out/r02_ozgemm_config4 python tools/prof_config4.py > gpurun_out/ncu_full.log 2>&1; echo ncu full rc=$?
python tools/ncu_summary.py gpurun_out/r02_ozgemm_config4.ncu-rep > gpurun_out/r02_ozgemm_config4_summary.txt 2>&1; cat gpurun_out/r02_ozgemm_config4_summary.txt
