mkdir -p gpurun_out
MLE_DGEMM_STAGE=bulk MLE_NVTX=1 timeout 3000 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_large.py::test_config5_full_size_on_one_gpu 2>&1 | tail -4
