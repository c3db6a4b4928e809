#!/bin/bash
# One GPU round-trip: gpu tests, phase timings at n=3600/16384, launch list at n=3600.
python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/pytest_gpu.txt
python tools/prof_eval.py 60 1 > gpurun_out/prof60.txt 2>&1
python tools/prof_eval.py 128 1 > gpurun_out/prof128.txt 2>&1
python tools/prof_eval.py 60 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_eval.py 60 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 290 > gpurun_out/launches_summary.txt
