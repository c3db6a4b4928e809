mkdir -p gpurun_out
cd paper_2601_11437_b200/csrc
cp linalg.cu /tmp/linalg_new.cu
cp ../../tools/ab_prev/linalg_prev.cu linalg.cu
make -B > /dev/null 2>&1 || echo OLD BUILD FAILED
cd ../..
python tools/stage_ab.py --child > gpurun_out/diag_old.txt 2>&1
python tools/stage_ab.py --child > gpurun_out/diag_old2.txt 2>&1
cp /tmp/linalg_new.cu paper_2601_11437_b200/csrc/linalg.cu
make -C paper_2601_11437_b200/csrc -B > /dev/null 2>&1 || echo NEW BUILD FAILED
python tools/stage_ab.py --child > gpurun_out/diag_new.txt 2>&1
python tools/stage_ab.py --child > gpurun_out/diag_new2.txt 2>&1
python - <<'PY'
import json
def load(f):
    for l in open(f):
        if l.startswith("RESULT "): return json.loads(l[7:])
    print(f, "NO RESULT", open(f).read()[-1500:]); return None
o, o2, n, n2 = (load('gpurun_out/diag_%s.txt' % k) for k in ('old', 'old2', 'new', 'new2'))
if o and n:
    print("bits config2 equal:", o["config2_bits"] == n["config2_bits"], " config3 equal:", o["config3_bits"] == n["config3_bits"])
    for k in ("config2_batched_loglik_ms", "config2_batched_eval_all_ms", "config3_eval_all_ms"):
        print(k, "old", round(o[k], 3), round(o2[k], 3), "new", round(n[k], 3), round(n2[k], 3))
    print("config3 potrf old", o["config3_phases"]["potrf_ms"], "new", n["config3_phases"]["potrf_ms"])
PY
timeout 900 python -m pytest tests/test_gpu_likelihood.py tests/test_gpu_fits.py -q -x 2>&1 | tail -2
