#!/bin/bash
python scripts/gemm_timeline.py 128 gu13 > gpurun_out/r2f_tl128.txt 2>&1
python scripts/gemm_timeline.py 8 > gpurun_out/r2f_tl8.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_kernels.py -q -x 2>&1 | tail -3 > gpurun_out/r2f_tests.log
cat gpurun_out/r2f_tests.log
