#!/bin/bash
timeout 600 compute-sanitizer --tool memcheck --show-backtrace no --print-limit 5 python scripts/gemm_timeline.py 128 > gpurun_out/dbg_memcheck.txt 2>&1
head -60 gpurun_out/dbg_memcheck.txt
