mkdir -p gpurun_out
base="-DMLE_DGEMM_STAGES_WIDE=3 -DMLE_DGEMM_STAGES_NARROW=2 -DMLE_DGEMM_BK_NARROW=16"
for dbg in 0 1 2 3; do
  make -C paper_2601_11437_b200/csrc -B EXTRA="$base -DMLE_DGEMM_DBG=$dbg" > /dev/null 2>&1 || echo BUILD FAILED
  echo "== dbg $dbg"
  for i in 1 2; do timeout 600 python -m pytest tests/test_gpu_likelihood.py -x -q 2>&1 | tail -2; done
done
