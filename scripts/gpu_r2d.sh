#!/bin/bash
python scripts/gemm_timeline.py 128 down13,gu13,qkv13 > gpurun_out/r2d_tl128.txt 2>&1
python scripts/gemm_timeline.py 32 down13,gu13 > gpurun_out/r2d_tl32.txt 2>&1
python -m pytest tests/test_gpu_headline.py -q -s 2>&1 | grep -E "headline greedy|passed|failed" > gpurun_out/r2d_headline.log
