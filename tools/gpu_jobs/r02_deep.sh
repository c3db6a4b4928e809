AB_VAR=MLE_INNER_DEEP timeout 600 python tools/boundary_ab.py
for f in 1 0; do echo "== deep $f"; MLE_INNER_DEEP=$f timeout 300 python tools/prof_batch.py 1 5 2>&1 | tail -1 | cut -c 1-170; done
timeout 600 python tools/diag_trace_probe.py > gpurun_out/diag_probe6.txt 2>&1; head -34 gpurun_out/diag_probe6.txt | tail -31
timeout 1200 python -m pytest tests/test_gpu_fits.py tests/test_gpu_likelihood.py tests/test_gpu_ozaki.py tests/test_gpu_nugget.py tests/test_gpu_two_sided.py tests/test_gpu_distributed.py -m gpu -q -x 2>&1 | tail -2
timeout 600 python tools/run_config.py config4 --breakdown-only 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('c4', d['loglik_phases_ms']['potrf_ms'], d['eval_all_phases_ms']['total_ms'])"
timeout 600 python tools/run_config.py config3 --breakdown-only 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('c3', d['loglik_phases_ms']['potrf_ms'], d['eval_all_phases_ms']['total_ms'])"
