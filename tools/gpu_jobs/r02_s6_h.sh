mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s6h.log 2>&1; echo smoke rc=$?
timeout 3000 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/gputest_s6h.log 2>&1; echo gputest rc=$?; tail -14 gpurun_out/gputest_s6h.log
