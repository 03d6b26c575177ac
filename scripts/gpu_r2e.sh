#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r2e_tests.log
python scripts/gemm_timeline.py 128 gu13,qkv13 > gpurun_out/r2e_tl128.txt 2>&1
python scripts/gemm_timeline.py 32 gu13 > gpurun_out/r2e_tl32.txt 2>&1
python scripts/gemm_timeline.py 8 > gpurun_out/r2e_tl8.txt 2>&1
python bench.py --steps 20 --warmup 5 --serve-horizon 0 --skip-cpu > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err
cat gpurun_out/r2e_tests.log
