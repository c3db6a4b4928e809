mkdir -p gpurun_out
python tools/stage_ab.py MLE_DGEMM_STAGE=cpasync MLE_DGEMM_STAGE=bulk MLE_DGEMM_STAGE=cpasync MLE_DGEMM_STAGE=bulk > gpurun_out/stage_ab.txt 2>&1
make -C paper_2601_11437_b200/csrc -B EXTRA="-DMLE_DGEMM_STAGES_WIDE=3 -DMLE_DGEMM_STAGES_NARROW=2 -DMLE_DGEMM_BK_NARROW=32" > /dev/null 2>&1 || echo BUILD FAILED
python tools/stage_ab.py MLE_DGEMM_STAGE=cpasync MLE_DGEMM_STAGE=bulk MLE_DGEMM_STAGE=cpasync MLE_DGEMM_STAGE=bulk > gpurun_out/stage_ab_s2.txt 2>&1
make -C paper_2601_11437_b200/csrc -B > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
