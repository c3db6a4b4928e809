for mb in 4 3 2; do
  make -C paper_2601_11437_b200/csrc -B EXTRA=-DMLE_GEN_MINB=$mb > /dev/null 2>&1
  grep -A2 "gen_engine_kernelILi1" paper_2601_11437_b200/csrc/ptxas.log | tail -2 | head -1
  echo "== MINB $mb (config 2, full storage)"; timeout 300 python tools/gen_bench.py 2>&1 | grep "gen GB/s" | tail -1
  echo "== MINB $mb (config 2 forced 2s: lower-only)"; MLE_SOLVE=2s timeout 300 python tools/gen_bench.py 2>&1 | grep "gen GB/s" | tail -1
done
make -C paper_2601_11437_b200/csrc -B > /dev/null 2>&1
