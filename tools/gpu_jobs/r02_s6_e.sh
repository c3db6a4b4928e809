mkdir -p gpurun_out
for st in bulk cpasync; do
  export MLE_DGEMM_STAGE=$st
  python tools/prof_eval.py 128 1 > /dev/null 2>&1 || echo run failed
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:dgemm_kernel -c 400 --csv --log-file gpurun_out/dg_$st.csv python tools/prof_eval.py 128 0 > /dev/null 2>&1
  IDX=$(python - <<PY
import csv
rows=[r for r in csv.DictReader(l for l in open('gpurun_out/dg_$st.csv') if l.startswith('"'))]
best=max(range(len(rows)), key=lambda i: float(rows[i]['Metric Value']))
print(best)
PY
)
  echo "$st: largest dgemm launch index $IDX"
  ncu --set full --clock-control none --import-source on -k regex:dgemm_kernel --launch-skip $IDX -c 1 -o gpurun_out/r02_dgemm_$st python tools/prof_eval.py 128 0 > /dev/null 2>&1
done
unset MLE_DGEMM_STAGE
ls -la gpurun_out/*.ncu-rep
