#!/bin/bash
# K1 split fill (CTAs per SM before splitting stops): decode rounds at serving batches
out=gpurun_out/r3r; mkdir -p $out
for rep in 1 2; do
for f in 4 8 16; do
  for b in 8 16 32; do
    MUX_K1_FILL=$f timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --serve-horizon 0 --skip-cpu --attn-steps 2 --e2e-steps 0 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'fill': $f, 'batch': $b, 'tok_s': d['value'], 'step_frac': d['step_roofline']['frac'], 'k1': d['roofline_secondary']['achieved'], 'mhz': d['clocks']['sm_mhz']}))" >> $out/rounds.jsonl
  done
done
done
cat $out/rounds.jsonl
