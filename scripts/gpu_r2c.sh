#!/bin/bash
# Round-2: re-run the previously failing GPU tests, GEMM timelines, C1 ablation.
python -m pytest tests/test_gpu_headline.py tests/test_gpu_tp_ipc.py tests/test_gpu_model.py -q -s -k "headline_decode_tokens or tp2" 2>&1 | tail -8 > gpurun_out/r2c_tests.log
python scripts/gemm_timeline.py 128 x > gpurun_out/r2_gemm_timeline.txt 2>&1
python scripts/gemm_timeline.py 32 > gpurun_out/r2_gemm_timeline_m32.txt 2>&1
python scripts/gemm_timeline.py 8 > gpurun_out/r2_gemm_timeline_m8.txt 2>&1
bash scripts/sched_ablation_c1.sh gpurun_out/sched_c1 > /dev/null 2>&1
tail -n 6 gpurun_out/sched_c1/summary.jsonl
cat gpurun_out/r2c_tests.log
