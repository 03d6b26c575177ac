import sys, json
sys.path.insert(0, ".")
from paper_2404_02015_b200 import calibrate
m = calibrate.measure("7b", decode_batches=(1,), decode_ctx=(128,), prefill_tokens=(256, 512, 1024, 1536, 2048, 3072, 4096), sm_granules=())
print(json.dumps(m["prefill"]))
