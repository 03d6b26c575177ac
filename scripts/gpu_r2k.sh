#!/bin/bash
# Round-2 re-entry check at HEAD: GPU suite, default bench, reference arm, ncu launch list
out=gpurun_out/r2k; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > $out/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/ref.json 2> $out/ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $out/launches.csv \
  python bench.py --steps 2 --warmup 3 --skip-cpu --serve-horizon 0 --e2e-steps 0 --attn-steps 0 > $out/ncu_bench.log 2>&1
gzip -f $out/launches.csv
tail -3 $out/tests.log; cat $out/smoke.log | tail -2; head -c 1500 $out/bench.json; echo; head -c 800 $out/ref.json
