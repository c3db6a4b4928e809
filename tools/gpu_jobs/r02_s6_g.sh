mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_seq_derivs.py -q -x 2>&1 | tail -3
timeout 300 python tools/run_config5_seq.py n=20000 gpurun_out/config5_seq_n20000.json > gpurun_out/c5_small.log 2>&1; echo small rc=$?; tail -3 gpurun_out/c5_small.log
timeout 2700 python tools/run_config5_seq.py fit gpurun_out/config5_seq_1gpu.json > gpurun_out/c5.log 2>&1; echo full rc=$?; tail -5 gpurun_out/c5.log
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
