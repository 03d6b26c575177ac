#!/bin/bash
# Round-2 GPU check: headline parity, the whole -m gpu suite, one bench run.
python -m pytest tests/test_gpu_headline.py -q -s 2>&1 | tail -30 > gpurun_out/r2_headline.log
python -m pytest tests -m gpu -q 2>&1 | tail -25 > gpurun_out/r2_gputests.log
[ "${1:-}" = "nobench" ] || python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
tail -n 3 gpurun_out/r2_headline.log gpurun_out/r2_gputests.log
