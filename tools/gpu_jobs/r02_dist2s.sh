timeout 1200 python -m pytest tests/test_gpu_distributed.py -m gpu -q -x > gpurun_out/gputest_dist2s.log 2>&1; echo rc=$?; tail -25 gpurun_out/gputest_dist2s.log
timeout 1500 python tools/dist_config4_check.py > gpurun_out/dist_config4_2s.json 2> gpurun_out/dist_config4_2s.err; echo rc=$?; python -c "
import json; d=json.load(open('gpurun_out/dist_config4_2s.json')); w=d['world2']; print(w['loglik_rel'], w['score_rel_scale'], w['fisher_rel'], w['seconds_sequential_ranks'], d['single']['seconds'])"
