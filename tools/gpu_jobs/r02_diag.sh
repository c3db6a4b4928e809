mkdir -p gpurun_out
rm -f gpurun_out/diag_pass_trace.txt
MLE_TRACE=gpurun_out/diag_pass_trace.txt timeout 600 python tools/diag_trace_probe.py > gpurun_out/diag_probe.txt 2>&1; echo probe rc=$?; cat gpurun_out/diag_probe.txt | head -60
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_lat tools/microbench/fp64_lat.cu && /tmp/fp64_lat > gpurun_out/fp64_lat.txt 2>&1; cat gpurun_out/fp64_lat.txt
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:gen_engine_kernel<1>" -c 1 -o gpurun_out/r02_gen_derivs_config4 python tools/prof_config4.py > gpurun_out/ncu_gen1.log 2>&1; echo ncu gen1 rc=$?
python tools/ncu_summary.py gpurun_out/r02_gen_derivs_config4.ncu-rep > gpurun_out/r02_gen_derivs_summary.txt 2>&1; cat gpurun_out/r02_gen_derivs_summary.txt
