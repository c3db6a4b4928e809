mkdir -p gpurun_out
for c in 124 96 72 48; do echo "== far cap $c"; MLE_FAR_CTAS=$c timeout 300 python tools/prof_batch.py 1 5 2>&1 | tail -2; done > gpurun_out/farcap_c2.txt
cat gpurun_out/farcap_c2.txt
for c in 124 96; do echo "== far cap $c config4"; MLE_FAR_CTAS=$c timeout 600 python tools/run_config.py config4 --breakdown-only 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['loglik_phases_ms']['potrf_ms'], d['eval_all_phases_ms']['total_ms'])"; done
