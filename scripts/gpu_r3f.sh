#!/bin/bash
# launch list at serving-shaped batch 16 (both models, whole-GPU streams)
out=gpurun_out/r3f; mkdir -p $out
CUDA_MODULE_LOADING=EAGER timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
  --log-file $out/launches_b16.csv python bench.py --batch 16 --steps 2 --warmup 3 --skip-cpu --serve-horizon 0 --e2e-steps 0 --attn-steps 0 \
  --partition-sms none > $out/ncu_b16.log 2>&1
python scripts/launch_summary.py $out/launches_b16.csv | head -12
gzip -f $out/*.csv
