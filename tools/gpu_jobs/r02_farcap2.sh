for c in 148 124 96 72 48; do echo "== far cap $c config2"; MLE_FAR_CTAS=$c timeout 300 python tools/prof_batch.py 1 5 2>&1 | tail -1 | cut -c 1-140; done
