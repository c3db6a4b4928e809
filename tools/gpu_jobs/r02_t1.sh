mkdir -p gpurun_out
timeout 600 python tools/prof_batch.py 1 5 2>&1 | tail -2
timeout 600 python tools/prof_batch.py 2 3 2>&1 | tail -1
timeout 600 python tools/diag_trace_probe.py > gpurun_out/diag_probe4.txt 2>&1; echo probe rc=$?; head -36 gpurun_out/diag_probe4.txt
timeout 1200 python -m pytest tests/test_gpu_fits.py tests/test_gpu_likelihood.py tests/test_gpu_distributed.py tests/test_gpu_ozaki.py tests/test_gpu_nugget.py -m gpu -q -x > gpurun_out/gputest_t1.log 2>&1; echo gputest rc=$?; tail -3 gpurun_out/gputest_t1.log
timeout 600 python tools/run_config.py config4 --breakdown-only 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('c4', d['loglik_phases_ms']['potrf_ms'], d['eval_all_phases_ms']['total_ms'])"
