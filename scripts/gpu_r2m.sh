#!/bin/bash
# ncu visibility diagnostics + small-batch step sweep (graphs on/off)
out=gpurun_out/r2m; mkdir -p $out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/diag_gemm_one.csv \
  python scripts/gemm_one.py 128 15360 5120 0 > $out/diag_gemm_one.log 2>&1
timeout 300 python scripts/gemm_micro.py 128 > $out/gemm_micro_128.txt 2>&1
timeout 300 python scripts/gemm_micro.py 16 > $out/gemm_micro_16.txt 2>&1
MUX_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $out/diag_bench_none.csv \
  -k regex:"gemm|decode_attention|kv_append|rmsnorm|argmax|embed|gather|scatter" \
  python bench.py --steps 2 --warmup 3 --skip-cpu --serve-horizon 0 --e2e-steps 0 --attn-steps 0 --partition-sms none > $out/diag_bench_none.log 2>&1
CUDA_MODULE_LOADING=EAGER MUX_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $out/diag_bench_eager.csv \
  python bench.py --steps 2 --warmup 3 --skip-cpu --serve-horizon 0 --e2e-steps 0 --attn-steps 0 --partition-sms none > $out/diag_bench_eager.log 2>&1
for g in 1 0; do
  for p in none auto; do
    for b in 8 16 32 64 128; do
      MUX_GRAPHS=$g timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --serve-horizon 0 --skip-cpu --attn-steps 2 --e2e-steps 0 --partition-sms $p 2>/dev/null \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'graphs': $g, 'part': '$p', 'batch': $b, 'tok_s': d['value'], 'ms': d['ms_per_step'], 'jobs': d['run']['job_ms_per_step'], 'step_frac': d['step_roofline']['frac'], 'gemm_gbs': d['roofline']['achieved'] if 'gemm' in d['roofline']['kernel'] else d['roofline_secondary']['achieved'], 'k1_gbs': d['roofline']['achieved'] if 'decode_att' in d['roofline']['kernel'] else d['roofline_secondary']['achieved'], 'mhz': d['clocks']['sm_mhz']}))" >> $out/rounds.jsonl
    done
  done
done
for f in $out/diag_*.log; do echo "== $f"; grep -E "ERROR|Profiling|No kernels" $f | sort | uniq -c | head -5; done
for f in $out/diag_*.csv; do echo "== $f"; python - "$f" <<'PY'
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r]
if hi:
    c = collections.Counter(r[4].split("(")[0] for r in rows[hi[0] + 1:] if len(r) > 5)
    print(c.most_common(12))
PY
done
gzip -f $out/*.csv
cat $out/rounds.jsonl; head -12 $out/gemm_micro_128.txt
