mkdir -p gpurun_out
timeout 600 python tools/prof_batch.py 1 5 2>&1 | tail -2
rm -f gpurun_out/diag_pass_trace.txt
MLE_TRACE=gpurun_out/diag_pass_trace.txt timeout 600 python tools/diag_trace_probe.py > gpurun_out/diag_probe3.txt 2>&1; echo probe rc=$?; head -20 gpurun_out/diag_probe3.txt
timeout 1200 python -m pytest tests/test_gpu_fits.py tests/test_gpu_likelihood.py tests/test_gpu_distributed.py -m gpu -q -x > gpurun_out/gputest_pdl.log 2>&1; echo gputest rc=$?; tail -3 gpurun_out/gputest_pdl.log
