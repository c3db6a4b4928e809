mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:gen_engine_kernel -c 8 -o gpurun_out/r02_gen_staged_config4 python tools/prof_config4.py > gpurun_out/ncu_gen_staged.log 2>&1; echo ncu gen rc=$?
python tools/ncu_summary.py gpurun_out/r02_gen_staged_config4.ncu-rep > gpurun_out/r02_gen_staged_summary.txt 2>&1; cat gpurun_out/r02_gen_staged_summary.txt
