mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:gen_engine_kernel<\(int\)1>" -c 1 -o gpurun_out/r02_gen_derivs_config4 python tools/prof_config4.py > gpurun_out/ncu_gen1.log 2>&1; echo ncu gen1 rc=$?
python tools/ncu_summary.py gpurun_out/r02_gen_derivs_config4.ncu-rep > gpurun_out/r02_gen_derivs_summary.txt 2>&1; cat gpurun_out/r02_gen_derivs_summary.txt
