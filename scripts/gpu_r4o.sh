#!/bin/bash
# last check at HEAD: GPU suite and smoke
out=gpurun_out/r4o; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q > $out/gpu_suite.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1
tail -n 1 $out/gpu_suite.log; tail -n 1 $out/smoke.log
