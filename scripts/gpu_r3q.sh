#!/bin/bash
# Final round-2 measurement at HEAD: GPU suite, smoke, full bench (serving + cpu baseline), reference arm, ncu launch list
out=gpurun_out/r3q; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q > $out/gpu_suite.log 2>&1
timeout 300 python -m pytest tests/test_gpu_headline.py -q -s -k tokens 2>&1 | grep -E "parity|passed|failed" > $out/headline_rate.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/ref.json 2> $out/ref.err
CUDA_MODULE_LOADING=EAGER timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
  --log-file $out/launches.csv python bench.py --steps 2 --warmup 3 --skip-cpu --serve-horizon 0 --e2e-steps 0 --attn-steps 0 \
  --partition-sms none > $out/ncu_launches.log 2>&1
gzip -f $out/launches.csv
tail -3 $out/gpu_suite.log; cat $out/headline_rate.log; tail -1 $out/smoke.log; head -c 600 $out/bench.json; echo
