mkdir -p gpurun_out
for c in 148 136 124; do echo "== far cap $c config4"; MLE_FAR_CTAS=$c timeout 600 python tools/run_config.py config4 --breakdown-only 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['loglik_phases_ms']['potrf_ms'], d['eval_all_phases_ms']['total_ms'])"; done
for c in 148 124; do echo "== far cap $c config2"; MLE_FAR_CTAS=$c timeout 300 python tools/prof_batch.py 1 5 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_gpu_two_sided.py -m gpu -q -x 2>&1 | tail -3
