#!/bin/bash
out=gpurun_out/r2j; mkdir -p $out
for g in 1 0; do
  MUX_GRAPHS=$g MUX_RT_TIMELINE=$out/tl_$g.csv python serve.py --rates 120,60 --horizon 3 --realtime 2>/dev/null | tail -1 > $out/serve_rt_$g.json
done
gzip -f $out/tl_*.csv
for f in $out/serve_rt_*.json; do echo $f; head -c 330 $f; echo; done
