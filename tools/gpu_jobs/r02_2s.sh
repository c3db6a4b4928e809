mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_two_sided.py -m gpu -q -x > gpurun_out/gputest_2s.log 2>&1; echo 2s rc=$?; tail -30 gpurun_out/gputest_2s.log
for t in 0 2; do OZ_NTILE=$t timeout 300 ./tools/oz_gemm_test 4 1 5; OZ_NTILE=$t timeout 300 ./tools/oz_gemm_test 1 1 5; done > gpurun_out/oz_grouped.txt 2>&1; grep -E "ozgemm|!!" gpurun_out/oz_grouped.txt
timeout 600 python tools/run_config.py config4 --breakdown-only --kernel-profile > gpurun_out/c4_grouped.json 2> gpurun_out/c4_grouped.err; echo c4 rc=$?; tail -c 1500 gpurun_out/c4_grouped.json
MLE_SOLVE=2s timeout 600 python tools/run_config.py config4 --breakdown-only --kernel-profile > gpurun_out/c4_2s.json 2> gpurun_out/c4_2s.err; echo c4 2s rc=$?; tail -c 1500 gpurun_out/c4_2s.json
