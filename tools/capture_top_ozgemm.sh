ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ozgemm_persistent -c 80 --csv --log-file gpurun_out/ozl.csv python tools/prof_batch.py 2 1 > /dev/null 2>&1
IDX=$(python - <<'PY'
import csv
rows=[r for r in csv.DictReader(l for l in open('gpurun_out/ozl.csv') if l.startswith('"'))]
best=max(range(len(rows)), key=lambda i: float(rows[i]['Metric Value']))
print(best)
PY
)
echo "largest ozgemm launch index $IDX"
ncu --set full --clock-control none --import-source on -k regex:ozgemm_persistent --launch-skip $IDX -c 1 -o gpurun_out/ozgemm_big python tools/prof_batch.py 2 1 > /dev/null 2>&1
ls gpurun_out/ozgemm_big*
