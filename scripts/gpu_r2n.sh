#!/bin/bash
# ncu launch list + full captures (eager loading, whole-GPU streams), racecheck
# control, bench --placement (2 ranks on one GPU), TP allreduce cost, serving timeline
out=gpurun_out/r2n; mkdir -p $out
export CUDA_MODULE_LOADING=EAGER
nvcc -gencode arch=compute_100a,code=sm_100a -o $out/bmc scripts/sanitizer/bulk_mbar_control.cu && \
  timeout 120 compute-sanitizer --tool racecheck $out/bmc > $out/san_control.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
  --log-file $out/launches.csv python bench.py --steps 2 --warmup 3 --skip-cpu --serve-horizon 0 --e2e-steps 0 --attn-steps 0 \
  --partition-sms none > $out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tn_kernel -s 300 -c 5 -o $out/gemm_full \
  python bench.py --steps 2 --warmup 3 --skip-cpu --serve-horizon 0 --e2e-steps 0 --attn-steps 0 --partition-sms none > $out/ncu_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attention -s 100 -c 1 -o $out/k1_full \
  python bench.py --steps 2 --warmup 3 --skip-cpu --serve-horizon 0 --e2e-steps 0 --attn-steps 0 --partition-sms none > $out/ncu_k1.log 2>&1
unset CUDA_MODULE_LOADING
timeout 900 python -m pytest tests/test_bench_placement.py -q -x -m gpu > $out/placement_test.log 2>&1
timeout 900 python scripts/tp_allreduce_cost.py $out/tp_allreduce.json > $out/tp_allreduce.log 2>&1
MUX_RT_TIMELINE=$out/tl_rt.csv timeout 600 python serve.py --rates 120,60 --horizon 3 --realtime > $out/serve_rt.json 2> $out/serve_rt.err
python scripts/rt_timeline.py $out/tl_rt.csv > $out/tl_rt_summary.txt 2>&1
gzip -f $out/*.csv
tail -3 $out/san_control.log; tail -3 $out/placement_test.log; tail -6 $out/tp_allreduce.log; head -c 600 $out/serve_rt.json; echo; head -30 $out/tl_rt_summary.txt
for f in $out/ncu_*.log; do echo "== $f"; grep -E "ERROR|No kernels" $f | head -3; done
