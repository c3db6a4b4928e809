mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_large.py -m gpu -q -k "distributed or panels or world or stream or window" > gpurun_out/gputest_dist.log 2>&1; echo gputest rc=$?; tail -30 gpurun_out/gputest_dist.log
