mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_two_sided.py -m gpu -q -x > gpurun_out/gputest_2s.log 2>&1; echo 2s rc=$?; tail -30 gpurun_out/gputest_2s.log
MLE_SOLVE=2s timeout 600 python tools/run_config.py config4 --breakdown-only --kernel-profile > gpurun_out/c4_2s.json 2> gpurun_out/c4_2s.err; echo c4 2s rc=$?; tail -c 1200 gpurun_out/c4_2s.json
