#!/bin/bash
# Round-2 check after the K3 flat-stream changes: GPU suite, smoke, full bench (serving + cpu baseline)
out=gpurun_out/r4g; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q > $out/gpu_suite.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err
tail -3 $out/gpu_suite.log; tail -1 $out/smoke.log; head -c 700 $out/bench.json; echo
python - <<'PY'
import json
b = json.loads(open("gpurun_out/r4g/bench.json").read().strip().splitlines()[-1])
print({k: b.get(k) for k in ("value", "ms_per_step")}, b["e2e"]["value"], b.get("step_roofline", {}).get("frac"), b.get("serving", {}).get("value"), b.get("clocks"), b.get("prefill"))
PY
