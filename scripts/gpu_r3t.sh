#!/bin/bash
out=gpurun_out/r3t; mkdir -p $out
for i in 1 2; do
timeout 600 python bench.py --skip-cpu --serve-horizon 0 > $out/bench_$i.json 2> $out/bench_$i.err
python -c "import json; d=json.load(open('$out/bench_$i.json')); print(d['value'], d['e2e']['value'], d['step_roofline']['frac'], d['clocks']['sm_mhz'])"
done
