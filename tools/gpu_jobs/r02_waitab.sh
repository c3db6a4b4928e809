build() { make -C paper_2601_11437_b200/csrc -B EXTRA="$1" > /dev/null 2>&1; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 $1 -o tools/oz_gemm_test tools/oz_gemm_test.cu paper_2601_11437_b200/csrc/linalg.cu paper_2601_11437_b200/csrc/ozaki.cu > /dev/null 2>&1; }
for v in "" "-DOZ_TEST_WAIT=1" "-DOZ_EARLY_WAIT=1" "-DOZ_EARLY_WAIT=1 -DOZ_TEST_WAIT=1"; do
  build "$v"
  echo "== variant [$v]"
  timeout 300 ./tools/oz_gemm_test 4 1 5 | grep -E "ozgemm|!!" | sed 's/.*ozgemm/ozgemm/'
  timeout 300 ./tools/oz_gemm_test 1 1 5 | grep -E "ozgemm|!!" | sed 's/.*ozgemm/ozgemm/'
  OZ_DIAG=1 timeout 300 ./tools/oz_gemm_test 4 1 3 2>&1 | grep -E "mode 0\)|mode 7\)"
done
build ""
