#!/bin/bash
# ncu launch lists of the decode round at batch 8 / 16 / 32 per model (pair GEMM at every decode tile)
out=gpurun_out/r4j; mkdir -p $out
for b in 8 16 32; do
CUDA_MODULE_LOADING=EAGER timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
  --log-file $out/launches_b$b.csv python bench.py --batch $b --steps 2 --warmup 3 --skip-cpu --serve-horizon 0 --e2e-steps 0 --attn-steps 0 \
  --partition-sms none > $out/ncu_b$b.log 2>&1
python scripts/launch_summary.py $out/launches_b$b.csv > $out/launches_b$b.txt 2>&1
head -4 $out/launches_b$b.txt
gzip -f $out/launches_b$b.csv
done
for b in 8 16 32; do
timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --serve-horizon 0 --skip-cpu --attn-steps 2 --e2e-steps 0 2>/dev/null \
  | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'batch': $b, 'tok_s': d['value'], 'step_frac': d['step_roofline']['frac'], 'gemm_stream': d['roofline']['achieved'], 'gemm_frac': d['roofline']['frac'], 'mhz': d['clocks']['sm_mhz']}))" >> $out/rounds.jsonl
done
cat $out/rounds.jsonl
