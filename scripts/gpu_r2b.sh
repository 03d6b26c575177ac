bash scripts/gpu_round2_check.sh nobench
python scripts/gemm_timeline.py 128 x > gpurun_out/r2_gemm_timeline.txt 2>&1
python scripts/gemm_timeline.py 32 > gpurun_out/r2_gemm_timeline_m32.txt 2>&1
bash scripts/sched_ablation_c1.sh gpurun_out/sched_c1 > /dev/null 2>&1
tail -n 6 gpurun_out/sched_c1/summary.jsonl
