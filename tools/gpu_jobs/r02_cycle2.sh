mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_c2.log 2>&1; echo gputest rc=$?; tail -15 gpurun_out/gputest_c2.log
timeout 600 python tools/run_config.py config4 --breakdown-only --kernel-profile > gpurun_out/c4_la.json 2> gpurun_out/c4_la.err; echo c4 rc=$?; python -c "
import json; d=json.load(open('gpurun_out/c4_la.json')); print({k: d[k] for k in d if 'phases' in k or 'wall' in k})"
for m in w 2s; do MLE_SOLVE=$m timeout 600 python tools/run_config.py config3 --breakdown-only --kernel-profile > gpurun_out/c3_$m.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/c3_$m.json')); print('$m', {k: d[k] for k in d if 'phases' in k or 'wall' in k})"; done
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c4b.json 2> gpurun_out/bench_c4b.err; echo bench rc=$?; tail -c 300 gpurun_out/bench_c4b.json
