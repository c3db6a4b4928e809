mkdir -p gpurun_out
timeout 600 python tools/boundary_ab.py
for f in 1 0; do echo "== split $f"; MLE_BOUNDARY_SPLIT=$f timeout 300 python tools/prof_batch.py 1 5 2>&1 | tail -1 | cut -c 1-160; done
timeout 600 python tools/diag_trace_probe.py > gpurun_out/diag_probe5.txt 2>&1; head -34 gpurun_out/diag_probe5.txt | tail -31
timeout 1200 python -m pytest tests/test_gpu_fits.py tests/test_gpu_likelihood.py tests/test_gpu_ozaki.py tests/test_gpu_nugget.py tests/test_gpu_two_sided.py -m gpu -q -x > gpurun_out/gputest_bs.log 2>&1; echo gputest rc=$?; tail -3 gpurun_out/gputest_bs.log
timeout 600 python tools/run_config.py config4 --breakdown-only 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('c4', d['loglik_phases_ms']['potrf_ms'], d['eval_all_phases_ms']['total_ms'])"
MLE_SOLVE=2s timeout 600 python tools/run_config.py config3 --breakdown-only 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('c3', d['loglik_phases_ms']['potrf_ms'], d['eval_all_phases_ms']['total_ms'])"
