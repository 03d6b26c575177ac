#!/bin/bash
# HEAD with stream-K pair prefill GEMMs: full GPU suite, serving A/B (MUX_GEMM_2SM_MIN_M 256 = old dispatch)
out=gpurun_out/r3i; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q > $out/gpu_suite.log 2>&1
tail -3 $out/gpu_suite.log
for mm in 1000 256; do
  MUX_GEMM_2SM_MIN_M=$mm timeout 900 python serve.py --rates 120,60 --horizon 6 --realtime 2>/dev/null | tail -1 \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'min_m': $mm, 'tok_s': d['value'], 'window': d['arrival_window']['tok_s'], 'ttft_ms': d['ttft_ms'], 'tpot_ms': d['tpot_ms'], 'makespan_s': d['makespan_s']}))" >> $out/serve.jsonl
  MUX_GEMM_2SM_MIN_M=$mm timeout 900 python serve.py --rates 20,10 --horizon 8 --realtime 2>/dev/null | tail -1 \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'min_m': $mm, 'rates': '20,10', 'tok_s': d['value'], 'window': d['arrival_window']['tok_s'], 'ttft_ms': d['ttft_ms'], 'tpot_ms': d['tpot_ms']}))" >> $out/serve.jsonl
done
cat $out/serve.jsonl
