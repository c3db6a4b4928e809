for v in "-DMLE_GEN_EXACT_NOINLINE=0" "" "-DMLE_GEN_MINB=5" "-DMLE_GEN_MINB=6"; do
  make -C paper_2601_11437_b200/csrc -B EXTRA="$v" > /dev/null 2>&1
  echo "== [$v] full storage: $(timeout 300 python tools/gen_bench.py 2>&1 | grep 'gen GB/s' | tail -1 | cut -c 1-40)"
  echo "== [$v] lower-only: $(MLE_SOLVE=2s timeout 300 python tools/gen_bench.py 2>&1 | grep 'gen GB/s' | tail -1 | cut -c 1-40)"
done
make -C paper_2601_11437_b200/csrc -B > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_likelihood.py tests/test_gpu_special.py -m gpu -q -x 2>&1 | tail -2
