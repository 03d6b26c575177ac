#!/bin/bash
# bench (headline + serving), ncu launch list, one --set full capture of 4 consecutive decode GEMMs
python bench.py --steps 20 --warmup 5 > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2500 --csv \
  --log-file gpurun_out/r2g_launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --attn-steps 0 --skip-cpu --serve-horizon 0 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/r2g_launches.csv > gpurun_out/r2g_launches.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tn_kernel -s 400 -c 4 -o gpurun_out/r2g_gemm \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --attn-steps 0 --skip-cpu --serve-horizon 0 --partition-sms none > /dev/null 2>&1
cat gpurun_out/r2g_launches.txt
