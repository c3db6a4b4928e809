mkdir -p gpurun_out
for t in 0 3 1 2; do echo "== ntile $t"; OZ_NTILE=$t timeout 300 ./tools/oz_gemm_test 4 1 5; OZ_NTILE=$t timeout 300 ./tools/oz_gemm_test 1 1 5; done > gpurun_out/oz_variants.txt 2>&1
for t in 0 3; do echo "== diag ntile $t"; OZ_DIAG=1 OZ_NTILE=$t timeout 300 ./tools/oz_gemm_test 4 1 3; done > gpurun_out/oz_diag.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fits.py tests/test_gpu_special.py tests/test_gpu_large.py -m gpu -q -k "not window" > gpurun_out/gputest3.log 2>&1; echo gputest rc=$?; tail -5 gpurun_out/gputest3.log
for tool in memcheck racecheck synccheck; do timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_$tool.log 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/sanitizer_$tool.log; done
cat gpurun_out/oz_variants.txt | grep -v "^$"
