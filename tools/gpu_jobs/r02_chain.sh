mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fits.py tests/test_gpu_likelihood.py tests/test_gpu_ozaki.py tests/test_gpu_nugget.py -m gpu -q -x > gpurun_out/gputest_chain.log 2>&1; echo gputest rc=$?; tail -3 gpurun_out/gputest_chain.log
rm -f gpurun_out/diag_pass_trace.txt
MLE_TRACE=gpurun_out/diag_pass_trace.txt timeout 600 python tools/diag_trace_probe.py > gpurun_out/diag_probe2.txt 2>&1; echo probe rc=$?; head -40 gpurun_out/diag_probe2.txt
timeout 600 python tools/prof_batch.py 1 5 2>&1 | tail -3
timeout 900 python tools/fit_paths_probe.py config4 > gpurun_out/fit_paths_config4.json 2> gpurun_out/fit_paths.err; echo fitpaths rc=$?; python -c "
import json; d=json.load(open('gpurun_out/fit_paths_config4.json')); print(d['same_counts'], d['theta_hat_rel_diff'], d['2s']['seconds'], d['w']['seconds'], d['2s']['grad_calls'], d['2s']['loglik_calls'])"
